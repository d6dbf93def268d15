mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "numeric or multirank or cxx" > gpurun_out/pytest_num.log 2>&1; tail -25 gpurun_out/pytest_num.log
timeout 600 python tools/probe_numeric.py > gpurun_out/probe_numeric.log 2>&1; cat gpurun_out/probe_numeric.log
