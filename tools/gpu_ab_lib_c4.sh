#!/bin/bash
# smoother colour passes at 128^3 and at C4 size of library variants libipmg<tag>.so
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for t in "$@"; do
  echo "== $t 128^3"
  AB_QUICK=1 IPMG_LIB=paper_2405_18982_b200/libipmg${t}.so timeout 300 python tools/ab_kernels.py 3 4 7 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,3) for k,v in d.items() if k.startswith('smooth') and 'dir' not in k})"
  echo "== $t C4"
  AB_COARSE=2,2,1 AB_QUICK=1 IPMG_LIB=paper_2405_18982_b200/libipmg${t}.so timeout 300 python tools/ab_kernels.py 3 4 8 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,3) for k,v in d.items() if k.startswith('smooth') and 'dir' not in k})"
done
