#!/bin/bash
# NEXT-4 tensor-core prototype: timing + ncu of both variants (tools/tc_proto.cu)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
./tools/tc_proto.bin > gpurun_out/tc_proto.json 2>&1; cat gpurun_out/tc_proto.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ffma2_pass|mma_pass" -s 3 -c 1 -o gpurun_out/prof_tc_ffma2 -f ./tools/tc_proto.bin > /dev/null 2>&1; timeout 600 ncu --set full --clock-control none --import-source on -k regex:mma_pass -s 2 -c 1 -o gpurun_out/prof_tc_mma -f ./tools/tc_proto.bin > gpurun_out/prof_tc.log 2>&1
tail -2 gpurun_out/prof_tc.log
