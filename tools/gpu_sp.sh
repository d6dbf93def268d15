mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "chi2 or fit or smoke or numeric or multirank or bench_scaling or bridge" -x 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:chi2_tile_kernel -o gpurun_out/prof_chi2_rec python tools/probe_rec_ncu.py > gpurun_out/ncu_rec.log 2>&1; tail -1 gpurun_out/ncu_rec.log
