#!/bin/bash
# One GPU call at the end of a session: tools/gpu_round2.sh (smoke, tests, bench, launch
# list, ncu --set full of the smoother and the fp64 operator), then the C3 sweep and the
# configs C1/C4/C5/throughput-vs-size.
TAG=${1:-final}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
bash tools/gpu_round2.sh $TAG
timeout 1500 python tools/sweep_c3.py --out gpurun_out/${TAG}_c3_sweep.jsonl > gpurun_out/${TAG}_c3.log 2>&1
tail -2 gpurun_out/${TAG}_c3.log
timeout 1800 python tools/configs.py --out gpurun_out/${TAG}_configs.jsonl > gpurun_out/${TAG}_configs.log 2>&1
tail -2 gpurun_out/${TAG}_configs.log
