cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for T in 0 8; do
IPMG_PAIR3_TY=$T AB_COARSE=2,2,1 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:smooth_pair3 -s 1 -c 1 python tools/prof_smooth.py 3 4 8 2>&1 | grep -E "dram__bytes_read|gpu__time|lts__t_sector" | head -6
done
