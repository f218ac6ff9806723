#!/bin/bash
# ncu --set full with source of the 3D k=4 pair smoother (colour 1) and the 3D k=4 fp64
# operator at 128^3 cells; exports the SASS source pages (per-instruction stall reasons)
# and the raw metric pages for offline analysis (tools/stall_phases.py).
#   gpurun --timeout 1500 -- 'bash tools/gpu_stalls.sh TAG'
TAG=${1:-st}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail -30 gpurun_out/build_${TAG}.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smooth_pair3 -s 2 -c 1 \
  -o gpurun_out/stall_smooth_${TAG} -f python tools/prof_smooth.py 3 4 7 > gpurun_out/stall_smooth_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vmult_kernel -s 2 -c 1 \
  -o gpurun_out/stall_vmult_${TAG} -f python tools/prof_vmult.py 3 4 7 > gpurun_out/stall_vmult_${TAG}.log 2>&1
for r in smooth vmult; do
  ncu -i gpurun_out/stall_${r}_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/stall_${r}_${TAG}_sass.csv 2>/dev/null
  ncu -i gpurun_out/stall_${r}_${TAG}.ncu-rep --page raw --csv > gpurun_out/stall_${r}_${TAG}_raw.csv 2>/dev/null
done
ls -la gpurun_out | tail
