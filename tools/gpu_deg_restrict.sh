#!/bin/bash
# Per-degree A/B of the residual + restriction (fp32 and fp64, C3 sizes): default build vs
# libipmg_or0.so (IPMG_OP3_RESTRICT=0, the restrict_kernel)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "2:2,1,1:8" "3:2,2,2:7" "4:2,2,1:7" "5:2,1,1:7" "6:2,2,2:6"; do
  k=${cfg%%:*}; rest=${cfg#*:}; co=${rest%%:*}; nl=${rest#*:}
  for t in "" _or0; do
    AB_QUICK=1 AB_COARSE=$co IPMG_LIB=paper_2405_18982_b200/libipmg$t.so timeout 300 python tools/ab_kernels.py 3 $k $nl 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('k=$k [$t]', round(d['restrict32_ms'],4), round(d.get('restrict64_ms',-1),4))"
  done
done
