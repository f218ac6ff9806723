cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
bash tools/ab_run.sh "_base _fsz _base _fsz" "2 7 10" "3 4 7" "3 3 7"
