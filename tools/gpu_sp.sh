# ncu of the shared-mean staged-tile kernel, dp only (10M x 100)
mkdir -p gpurun_out
O=gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:shared_p_tma -s 10 -c 1 -o $O/prof_sp_tma_dp python tools/probe_shared_p.py 5 100 10000000 > /dev/null 2>&1
python tools/ncu_summary.py $O/prof_sp_tma_dp.ncu-rep
