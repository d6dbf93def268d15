mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "fit or smoke or multirank or bench_scaling or bridge" -x 2>&1 | grep -E "^E |passed|failed|Error" | head
timeout 300 python tools/probe_fit_launches.py 400
timeout 300 python -c "
import json, bench
d = bench.bench_fit_1e6(0); print(d['gd_armijo'], d['newton_numeric_hessian']['fit_iterations_per_s'])"
