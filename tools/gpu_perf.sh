mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log | grep -v "^\.\.\.\."
timeout 300 python tools/probe_chi2.py 100000000 2>&1 | tail -4
timeout 600 python tools/probe_numeric.py 2>&1 | tail -12
