#!/bin/bash
# A/B of environment switches on the 3D k=4 smoother: bash tools/gpu_ab_env.sh "ENV=a ENV2=b" "ENV=c" ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for envs in "$@"; do
  echo "== $envs"
  env $envs AB_QUICK=1 timeout 300 python tools/ab_kernels.py 3 4 7 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,3) for k,v in d.items() if k.startswith('smooth')})"
done
