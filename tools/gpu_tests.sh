cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_dist.log 2>&1
tail -30 gpurun_out/pytest_dist.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_par.log 2>&1
tail -5 gpurun_out/pytest_par.log
