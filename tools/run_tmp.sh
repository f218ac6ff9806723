cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
bash tools/ab_run.sh "_eig _rows _eig _rows" "2 7 10" "3 4 7" "3 3 7" "2 3 10"
