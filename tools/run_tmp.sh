cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hermite or clamped" > gpurun_out/pytest_herm.log 2>&1; tail -30 gpurun_out/pytest_herm.log
