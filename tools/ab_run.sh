#!/bin/bash
# A/B of library variants: bash tools/ab_run.sh "tag1 tag2 ..." "dim k levels" ["dim k levels" ...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAGS="$1"; shift
for cfg in "$@"; do
  for t in $TAGS; do
    IPMG_LIB=paper_2405_18982_b200/libipmg${t}.so timeout 300 python tools/ab_kernels.py $cfg 2>&1 | tail -1
  done
done
