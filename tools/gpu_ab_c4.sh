#!/bin/bash
# smoother colour passes at the C4 size (3D k=4, 256x256x128) under environment variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for envs in "$@"; do
  echo "== $envs"
  env $envs AB_COARSE=2,2,1 AB_QUICK=1 timeout 300 python tools/ab_kernels.py 3 4 8 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,3) for k,v in d.items() if k.startswith('smooth') and 'dir' not in k})"
done
