#!/bin/bash
# Per-degree A/B of one tools/ab_kernels.py timing key (C3 sizes): default build vs libipmg<TAG>.so
#   bash tools/gpu_deg_key.sh TAG KEY [KEY2]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; KEY=$2; KEY2=${3:-$2}
for cfg in "2:2,1,1:8" "3:2,2,2:7" "4:2,2,1:7" "5:2,1,1:7" "6:2,2,2:6"; do
  k=${cfg%%:*}; rest=${cfg#*:}; co=${rest%%:*}; nl=${rest#*:}
  for t in "" $TAG; do
    AB_QUICK=1 AB_COARSE=$co IPMG_LIB=paper_2405_18982_b200/libipmg$t.so timeout 300 python tools/ab_kernels.py 3 $k $nl 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('k=$k [$t]', round(d['$KEY'],4), round(d['$KEY2'],4))"
  done
done
