mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -30 gpurun_out/pytest_gpu.log | grep -v "^\.\.\.\."
./oracle/_ref/bridge_check gpu 2>&1 | tail -22
