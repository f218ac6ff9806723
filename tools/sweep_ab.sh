#!/bin/bash
# C3 sweep per library variant: bash tools/sweep_ab.sh "tag1 tag2" "1,2,3"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for t in $1; do
  IPMG_LIB=paper_2405_18982_b200/libipmg${t}.so timeout 900 python tools/sweep_c3.py --degrees $2 --out gpurun_out/sweep${t}.jsonl > gpurun_out/sweep${t}.log 2>&1
done
