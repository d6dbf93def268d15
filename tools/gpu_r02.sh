# Round-2 measurement pass on one B200: measured FP64 peak, the GPU suite,
# smoke, every bench line (both arms, the chi2 line, the self-spawned 2-rank
# path), the launch list and ncu captures of the dominant kernel of each config.
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > $O/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu.txt
./build/fp64_peak 0 5 > $O/fp64_peak.json 2>&1; cat $O/fp64_peak.json
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench_ours.json 2> $O/bench_ours.err; tail -2 $O/bench_ours.err
timeout 900 python bench.py --workload chi2 > $O/bench_chi2.json 2> $O/bench_chi2.err; tail -2 $O/bench_chi2.err
timeout 600 python bench.py --workload fit > $O/bench_fit.json 2> $O/bench_fit.err; tail -2 $O/bench_fit.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -2 $O/bench_ref.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --no-e2e --no-cpu-baseline --steps 5 > $O/bench_2rank.json 2> $O/bench_2rank.err; tail -2 $O/bench_2rank.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --no-parity > $O/launches_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_chi2.csv python tools/probe_chi2.py 100000000 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chi2_tile -s 3 -c 1 -o $O/prof_chi2 python tools/probe_chi2.py 100000000 5 > $O/ncu_chi2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd -s 3 -c 1 -o $O/prof_gaussnd python bench.py --steps 1 --warmup 3 --no-e2e --no-configs --no-cpu-baseline --no-parity > $O/ncu_gaussnd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd -s 3 -c 1 -o $O/prof_nd1000 python bench.py --workload gaussnd1000 --steps 1 --warmup 3 --no-e2e --no-configs --no-cpu-baseline --no-parity > $O/ncu_nd1000.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gauss_grad -s 3 -c 1 -o $O/prof_gauss1d python bench.py --workload gauss1d --steps 1 --warmup 3 --no-e2e --no-configs --no-cpu-baseline --no-parity > $O/ncu_gauss1d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adc_kernel_k_looped -s 2 -c 1 -o $O/prof_jit_looped python tools/probe_jit.py k_looped > $O/ncu_jit.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adc_kernel_k_rational -s 2 -c 1 -o $O/prof_jit_rational python tools/probe_jit.py k_rational > $O/ncu_jit2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gaussnd -s 3 -c 1 python tools/probe_gaussnd_variants.py 100 10000001 0 > $O/ncu_nd_odd.txt 2>&1
# kernel-level timings outside the bench: K2 over layouts and dims (auto vs the
# static schedule), the shared-mean forms
{
  for cfg in "100 10000000" "100 10000001" "100 10000010" "1000 1000000" "1000 1000003" \
             "2 400000000" "2 400000001" "8 100000000" "8 100000001" "37 27000001" "200 5000001" "300 3333334"; do
    timeout 300 python tools/probe_gaussnd_variants.py $cfg 0,100 2>&1 | tail -2 | sed "s/^/[$cfg] /"
  done
  for cfg in "100 10000000" "200 5000000" "37 27000000" "24 40000000" "16 60000000" "8 120000000" "2 480000000"; do
    timeout 300 python tools/probe_shared_p.py 9 $cfg 2>&1 | tail -2 | cut -c1-60 | sed "s/^/[shared-mean $cfg] /"
  done
} > $O/probes.txt 2>&1
python tools/ncu_summary.py $O/prof_*.ncu-rep > $O/ncu_summary.txt 2>&1
python tools/ncu_fp64_per_unit.py $O/prof_chi2.ncu-rep 1e8 >> $O/ncu_summary.txt 2>&1
for f in $O/prof_*.ncu-rep; do case "$f" in *prof_chi2.ncu-rep) ;; *) rm -f "$f";; esac; done
du -sh $O
