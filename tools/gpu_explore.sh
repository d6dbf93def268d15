# Exploration pass: gauss1d kernel-only timing, dim-1000 variants + ncu,
# shared-p with dx + ncu.
mkdir -p gpurun_out
timeout 300 python -c "
import json, bench
print(json.dumps(bench.bench_points_small(0, 'gauss1d')))
print(json.dumps(bench.bench_points_small(0, 'gaussnd1000')))
" 2>&1 | tail -2
timeout 300 python tools/probe_gaussnd_variants.py 1000 1000000 0,2,7,3 2>&1 | tail -4
timeout 300 python tools/probe_shared_p.py 2>&1 | tail -2
ADC_SHAREDP_STAGE=0 timeout 300 python tools/probe_shared_p.py 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd_tile -c 1 -o gpurun_out/prof_nd1000 python tools/probe_gaussnd_variants.py 1000 1000000 0 > gpurun_out/ncu_nd1000.log 2>&1; tail -1 gpurun_out/ncu_nd1000.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd_shared_p_kernel -c 1 -o gpurun_out/prof_spdx python tools/probe_shared_p.py > gpurun_out/ncu_spdx.log 2>&1; tail -1 gpurun_out/ncu_spdx.log
