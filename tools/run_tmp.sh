cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "2 7 8" "2 7 9" "2 7 10"; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_issued.avg.pct_of_peak_sustained_active --cache-control none --clock-control none -k regex:smooth_kernel -s 4 -c 2 python tools/prof_smooth.py $cfg 2>&1 | grep -E "smooth_kernel|gpu__time|dram__bytes|inst_exec|inst_issued" 
done
