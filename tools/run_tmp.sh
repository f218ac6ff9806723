cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python tools/table1_gpu.py --kernel clamped --levels 2,3,4,5,6 --forward-post --fp64 > gpurun_out/table2_clamped_fwd64.jsonl 2>&1
timeout 900 python tools/table1_gpu.py --kernel clamped --levels 2,3,4,5,6 --forward-post > gpurun_out/table2_clamped_fwd.jsonl 2>&1
