mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "fit or smoke or bridge or numeric or scaling" -x 2>&1 | grep -E "^E |passed|failed|Error" | head -20
