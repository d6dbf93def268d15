for t in 0 6 0 6; do ADC_CHI2_TUNE=$t timeout 300 python tools/probe_rec.py 2>&1 | grep -E "mode 2" | tail -1 | sed "s/^/tune=$t /"; done
python - <<'PY'
import os, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2203_06139_b200 as adc
from paper_2203_06139_b200 import synth
res = {}
for t in ("0", "6"):
    os.environ["ADC_CHI2_TUNE"] = t
    h = adc.sample_histogram("gpoly", synth.GPOLY_TRUTH, 10**7, -5.0, 5.0, 1e9, seed=7, zero_every=100)
    pl = adc.Chi2Plan("gpoly", 6, h)
    pl.set_precision(2)
    res[t] = np.array(pl.gradient(list(synth.GPOLY_INIT))[0]).tobytes()
print("bits equal:", res["0"] == res["6"])
PY
