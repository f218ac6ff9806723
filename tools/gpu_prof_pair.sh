#!/bin/bash
# ncu --set full (with source) of the 3D k=4 pair-kernel colour passes (colour 0 zero start, colour 1)
TAG=${1:-pp}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail -30 gpurun_out/build_${TAG}.log; exit 1; }
IPMG_PAIR3=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:smooth_pair3 -s 1 -c 2 \
  -o gpurun_out/prof_${TAG} -f python tools/prof_smooth.py 3 4 7 > gpurun_out/prof_${TAG}.log 2>&1
tail -3 gpurun_out/prof_${TAG}.log
