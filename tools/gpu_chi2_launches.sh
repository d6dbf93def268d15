# Per-kernel device times of the chi2 gradient pass (ncu launch list).
O=gpurun_out; mkdir -p $O
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_chi2.csv python tools/probe_chi2.py ${CHI2_BINS:-100000000} 3 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_chi2.csv")))
h = None; t = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r: h = r; continue
    if h and len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        t[r[h.index("Kernel Name")][:70]].append(float(r[h.index("Metric Value")]))
for k, v in t.items(): print(f"{len(v):3d} x {sum(v)/len(v)/1e3:8.2f} us  {k}")
PY
