import sys, time, json
sys.path.insert(0, ".")
import bench
print(json.dumps(bench.bench_fit_1e6(0))[:1500])
