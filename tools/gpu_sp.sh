mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "chi2 or fit or smoke or numeric or multirank or bench_scaling or bridge or recurrence" -x 2>&1 | grep -E "^E |passed|failed" | head
timeout 300 python tools/probe_fit_launches.py 400
timeout 300 python -c "
import json, bench
d = bench.bench_fit_1e6(0); print(d['gd_armijo']['fit_iterations_per_s'], d['newton_numeric_hessian']['fit_iterations_per_s'])"
