bash tools/gpu_chi2_alts.sh > /dev/null 2>&1
M=gpu__time_duration.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio
for rep in 1 2; do
echo "base: $(ncu --metrics $M --clock-control none -k regex:chi2_tile -s 5 -c 5 python tools/probe_chi2.py 100000000 10 2>/dev/null | grep -E 'duration|barrier|fp64|wait' | awk '{print $1, $NF}' | sort | awk '{a[$1]=a[$1]" "$2} END {for (k in a) print k, a[k]}')"
echo "barrier: $(cd /tmp/alt_barrier && ncu --metrics $M --clock-control none -k regex:chi2_tile -s 5 -c 5 python tools/probe_chi2.py 100000000 10 2>/dev/null | grep -E 'duration|barrier|fp64|wait' | awk '{print $1, $NF}' | sort | awk '{a[$1]=a[$1]" "$2} END {for (k in a) print k, a[k]}')"
done
