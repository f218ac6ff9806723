#!/bin/bash
# vmult (fp64/fp32), restriction, smoother of library variants (libipmg<tag>.so) over 3D degrees
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "3 2 7" "3 3 7" "3 4 7" "3 5 6" "3 6 6" "3 7 6"; do
  for t in "$@"; do
    echo "== $cfg $t"
    AB_QUICK=1 IPMG_LIB=paper_2405_18982_b200/libipmg${t}.so timeout 300 python tools/ab_kernels.py $cfg 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,3) for k,v in d.items() if k in ('vmult64_ms','vmult32_ms','restrict32_ms','smooth_c1_ms')})"
  done
done
