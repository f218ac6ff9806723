#!/bin/bash
# One GPU call: ncu --set full with source of the 3D k=4 fp32 smoother colour pass
# (shifted colour) and the fp64 3D k=4 operator; exports the SASS source pages.
#   gpurun --timeout 1200 -- 'bash tools/gpu_srcprof.sh TAG'
TAG=${1:-src}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smooth_kernel -s 4 -c 2 \
  -o gpurun_out/src_smooth_${TAG} -f python tools/prof_smooth.py 3 4 7 > gpurun_out/src_smooth_${TAG}.log 2>&1
ncu -i gpurun_out/src_smooth_${TAG}.ncu-rep --page source --csv --print-source sass --launch-skip 1 --launch-count 1 \
  > gpurun_out/src_smooth_${TAG}_sass.csv 2>/dev/null
ncu -i gpurun_out/src_smooth_${TAG}.ncu-rep --page source --csv --print-source cuda --launch-skip 1 --launch-count 1 \
  > gpurun_out/src_smooth_${TAG}_cuda.csv 2>/dev/null
ls -la gpurun_out
