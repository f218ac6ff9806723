cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -x -q -k "dirichlet" > gpurun_out/pytest_dir.log 2>&1; tail -30 gpurun_out/pytest_dir.log
