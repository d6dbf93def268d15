mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "fit or smoke or bridge or batch or multirank or recurrence or numeric" -x 2>&1 | grep -E "^E |passed|failed|Error" | head -20
timeout 300 python -c "
import json, bench
d = bench.bench_fit_1e6(0); print(d['gd_armijo']['fit_iterations_per_s'], d['newton_numeric_hessian'])"
