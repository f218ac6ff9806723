#!/bin/bash
# op3 (staged fp64 3D operator) check: GPU parity tests touching the fp64 operator, then
# A/B timing IPMG_OP3=0/1 of the operator and the solve (3D k=4, 128^3 cells)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-op3}
timeout 900 python -m pytest tests -m gpu -x -q -k "vmult or cg or fullsize or smoke or distributed or properties" > gpurun_out/${TAG}_pytest.txt 2>&1
tail -3 gpurun_out/${TAG}_pytest.txt
for rep in 1 2; do
  for o in 0 1; do
    echo "== IPMG_OP3=$o rep $rep"
    IPMG_OP3=$o timeout 300 python tools/ab_kernels.py 3 4 7 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(v,4) if isinstance(v,float) else v) for k,v in d.items() if k in ('vmult64_ms','solve_ms','iterations')})"
  done
done
