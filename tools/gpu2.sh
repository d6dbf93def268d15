mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 300 python tools/probe_kernels.py 2>&1 | grep -E "gaussnd|chi2|gauss1d"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; tail -c 3000 gpurun_out/bench_ours.json; tail -5 gpurun_out/bench_ours.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd -s 1 -c 1 -o gpurun_out/prof_gaussnd python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chi2_tile -s 2 -c 1 -o gpurun_out/prof_chi2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; tail -3 gpurun_out/ncu2.log
ls -la gpurun_out
