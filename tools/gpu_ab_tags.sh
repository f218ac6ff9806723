#!/bin/bash
# A/B of pair-kernel library variants libipmg<tag>.so ("" = the default build) on 3D k=4
# (128^3 cells): colour-pass times, each variant run twice in alternation.
#   gpurun -- 'bash tools/gpu_ab_tags.sh "" _rs _x'
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2; do
  for t in "$@"; do
    echo "== [$t] rep $rep"
    AB_QUICK=1 IPMG_LIB=paper_2405_18982_b200/libipmg${t}.so timeout 300 python tools/ab_kernels.py 3 4 7 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,4) for k,v in d.items() if k.startswith('smooth_c')})"
  done
done
