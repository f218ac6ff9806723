#!/bin/bash
# Per-degree A/B of the staged kernels (C3 sizes, 3D): fp64 operator IPMG_OP3=0/1 and fp32
# colour passes IPMG_PAIR3=0/1 (the environment forces the kernel on/off for every degree)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in "2:2,1,1:8" "3:2,2,2:7" "5:2,1,1:7" "6:2,2,2:6" "7:2,2,2:6" "4:2,2,1:7"; do
  k=${cfg%%:*}; rest=${cfg#*:}; co=${rest%%:*}; nl=${rest#*:}
  for o in 0 1; do
    echo "== k=$k OP3=$o PAIR3=$o"
    IPMG_OP3=$o IPMG_PAIR3=$o AB_QUICK=1 AB_COARSE=$co timeout 300 python tools/ab_kernels.py 3 $k $nl 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(v,4) if isinstance(v,float) else v) for k,v in d.items() if k in ('ndofs','vmult64_ms','smooth_c1_ms','smooth_c3_ms')})"
  done
done
