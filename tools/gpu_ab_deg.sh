#!/bin/bash
# pair kernel on/off per 3D degree (smoother colour passes), and the 3D parity tests with it forced on
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IPMG_PAIR3=1 timeout 900 python -m pytest tests -m gpu -x -q -k "d3 and (smoother or vcycle or cg or distributed or fullsize)" > gpurun_out/pytest_pair_all.log 2>&1; tail -3 gpurun_out/pytest_pair_all.log
for cfg in "3 2 7" "3 3 7" "3 4 7" "3 5 6" "3 6 6" "3 7 6"; do
  for P in 0 1; do
    echo "== $cfg PAIR3=$P"
    IPMG_PAIR3=$P AB_QUICK=1 timeout 300 python tools/ab_kernels.py $cfg 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,3) for k,v in d.items() if k in ('smooth_c1_ms','smooth_c3_ms','smooth_step_ms')})"
  done
done
