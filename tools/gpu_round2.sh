#!/bin/bash
# One GPU call (round 2): smoke, parity tests, bench line (C4 headline), ncu launch list of
# one C4 solve, ncu --set full of the finest-level smoother colour pass and the fp64 vmult.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round2.sh TAG'
TAG=${1:-r02}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
tail -2 gpurun_out/smoke_${TAG}.log
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1
tail -3 gpurun_out/pytest_gpu_${TAG}.log
fi
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
cat gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/bench_${TAG}.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
  --csv --log-file gpurun_out/launches_${TAG}.csv python profiles/solve_once.py > gpurun_out/launches_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smooth_pair3 -s 0 -c 2 \
  -o gpurun_out/prof_smooth_${TAG} -f python profiles/solve_once.py > gpurun_out/prof_smooth_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"op3_kernel|vmult_kernel" -s 0 -c 1 \
  -o gpurun_out/prof_vmult_${TAG} -f python profiles/solve_once.py > gpurun_out/prof_vmult_${TAG}.log 2>&1
fi
ls -la gpurun_out
