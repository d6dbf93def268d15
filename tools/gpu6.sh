mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
./oracle/_ref/bridge_check gpu | tail -14
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_ours.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['secondary'])"; tail -3 gpurun_out/bench_ours.err
