#!/bin/bash
# ncu --set full with source of the op3 fp64 operator (3D k=4, 128^3 cells) + A/B of variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-op3}
shift
for t in "" "$@"; do
  for rep in 1 2; do
    echo "== [$t] rep $rep"
    AB_QUICK=1 IPMG_LIB=paper_2405_18982_b200/libipmg${t}.so timeout 300 python tools/ab_kernels.py 3 4 7 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,4) for k,v in d.items() if k in ('vmult64_ms','restrict32_ms','smooth_c1_ms')})"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:op3_kernel -s 2 -c 1 \
  -o gpurun_out/prof_${TAG} -f python tools/prof_vmult.py 3 4 7 > gpurun_out/prof_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${TAG}_sass.csv 2>/dev/null
tail -2 gpurun_out/prof_${TAG}.log
