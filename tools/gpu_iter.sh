#!/bin/bash
# Quick GPU iteration: build, a pytest -m gpu subset, A/B of the 3D k=4 smoother
# (IPMG_PAIR3=0 legacy kernel vs 1 pair kernel) on the C3-sized level (128^3 cells).
#   gpurun --timeout 1500 -- 'bash tools/gpu_iter.sh TAG "pytest -k expr"'
TAG=${1:-it}
KEXPR=${2:-"d3k4 or distributed"}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail -30 gpurun_out/build_${TAG}.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > gpurun_out/pytest_${TAG}.log 2>&1
tail -15 gpurun_out/pytest_${TAG}.log
for P in 0 1; do
  IPMG_PAIR3=$P AB_QUICK=1 timeout 300 python tools/ab_kernels.py 3 4 7 > gpurun_out/ab_${TAG}_p$P.json 2>&1
  echo "PAIR3=$P"; cat gpurun_out/ab_${TAG}_p$P.json | tail -2
done
