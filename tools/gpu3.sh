mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/probe_kernels.py 2>&1 | grep -E "gaussnd|chi2|gauss1d"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chi2_tile -s 2 -c 1 -o gpurun_out/prof_chi2b python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; tail -2 gpurun_out/ncu2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussnd -s 1 -c 1 -o gpurun_out/prof_gaussnd_b python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu1.log 2>&1; tail -2 gpurun_out/ncu1.log
