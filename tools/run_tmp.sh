cd "${GRAFT_REPO_ROOT:-/root/repo}"
IPMG_LIB=paper_2405_18982_b200/libipmg_tma.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "smoother or vcycle or cg" 2>&1 | tail -2
bash tools/ab_run.sh "_notma _tma _notma _tma" "2 7 10" "3 4 7" "3 3 7"
