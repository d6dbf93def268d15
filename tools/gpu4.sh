mkdir -p gpurun_out
timeout 300 python tools/probe_chi2.py 100000000 2>&1 | tail -10
