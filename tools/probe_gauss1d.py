"""BASELINE configs[0] on the device: the Listing-1 kernel over 1M points,
timed as bench.py's cfg1 record does (the kernel alone from CUDA graphs with
a clean-L2 flush), plus the public-API time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.config_points("gauss1d", 0)
print(json.dumps({k: r[k] for k in ("kernel_ms", "api_ms", "value")} |
                 {"frac": r["roofline"]["frac"], "parity_ok": r["parity"]["ok"]}))
