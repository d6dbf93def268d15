# Full round-end style verification on one B200: tests, smoke, bench (both arms),
# launch list and ncu captures of the dominant kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt; ldd --version | head -1 >> gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
./oracle/_ref/bridge_check gpu > gpurun_out/bridge_gpu.log 2>&1; tail -1 gpurun_out/bridge_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -3 gpurun_out/bench_ours.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd_ -s 3 -c 1 -o gpurun_out/prof_gaussnd python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chi2_tile -s 3 -c 1 -o gpurun_out/prof_chi2 python tools/probe_chi2.py 100000000 0 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adc_kernel -s 2 -c 1 -o gpurun_out/prof_jit python tools/probe_jit.py > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:shared_p_tma -s 2 -c 1 -o gpurun_out/prof_sharedp python tools/probe_shared_p.py > gpurun_out/ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:shared_p_vec2 -s 2 -c 1 -o gpurun_out/prof_spv python tools/probe_shared_p.py > gpurun_out/ncu6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd_tile -c 1 -o gpurun_out/prof_nd1000 python tools/probe_gaussnd_variants.py 1000 1000000 0 > gpurun_out/ncu7.log 2>&1
# (kernels inside a graph with a conditional node cannot be profiled: the host loop runs the same multi kernel)
ADC_PROBE_HOST_LOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:chi2_multi -s 20 -c 1 -o gpurun_out/prof_multi python tools/probe_fit_1e6.py > gpurun_out/ncu5.log 2>&1
ls gpurun_out
# summaries here (the box's ncu), then drop the big reports so gpurun_out/
# stays under the 64 MiB copy-back limit (keep the two headline captures)
python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > gpurun_out/ncu_summary.txt 2>&1
python tools/ncu_fp64_per_unit.py gpurun_out/prof_chi2.ncu-rep 1e8 >> gpurun_out/ncu_summary.txt 2>&1
for f in gpurun_out/prof_*.ncu-rep; do case "$f" in *prof_gaussnd.ncu-rep|*prof_chi2.ncu-rep) ;; *) rm -f "$f";; esac; done
du -sh gpurun_out
