mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-e2e > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo "rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_2rank_gloo.json').read().strip().splitlines()[-1]); print('2-rank:', d['n_gpus'], d['value'], d['secondary'][0])"; tail -3 gpurun_out/bench_2rank_gloo.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gauss_grad_vec2 -s 5 -c 1 -o gpurun_out/prof_gauss1d python bench.py --workload gauss1d --steps 2 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu3.log 2>&1; tail -1 gpurun_out/ncu3.log
