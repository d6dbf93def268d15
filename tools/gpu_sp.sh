# ncu of the shared-mean staged-tile kernel (dp only and with dx, 10M x 100)
mkdir -p gpurun_out
O=gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:shared_p_tma -s 2 -c 1 -o $O/prof_sp_tma_dx python tools/probe_shared_p.py 3 100 10000000 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:shared_p_tma -s 5 -c 1 -o $O/prof_sp_tma_dp python tools/probe_shared_p.py 3 100 10000000 > /dev/null 2>&1
python tools/ncu_summary.py $O/prof_sp_tma_*.ncu-rep
