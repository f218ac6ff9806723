#!/bin/bash
# compute-sanitizer over every kernel (tools/sanitize.py): memcheck, racecheck, synccheck,
# initcheck; the legacy 3D smoother and the patch-pair smoother (IPMG_PAIR3=0 / 1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for P in 0 1; do
    Q=""; [ "$tool" = "racecheck" ] && Q="--quick"
    [ "$tool" = "initcheck" ] && Q="--quick"
    echo "== $tool IPMG_PAIR3=$P $Q"
    IPMG_PAIR3=$P timeout 1500 $CS --tool $tool --print-limit 20 python tools/sanitize.py $Q > gpurun_out/san_${tool}_p$P.log 2>&1
    echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|done|Error" gpurun_out/san_${tool}_p$P.log | tail -4
  done
done
