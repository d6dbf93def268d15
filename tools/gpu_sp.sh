mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "shared_p or smoke" -x 2>&1 | tail -1
for rep in 1 2; do
ADC_SHAREDP_VEC=1 timeout 300 python tools/probe_shared_p.py 2>&1 | tail -2 | head -1
ADC_SHAREDP_VEC=0 ADC_SHAREDP_TMA=1 timeout 300 python tools/probe_shared_p.py 2>&1 | tail -2
ADC_SPT_V16=1 ADC_SHAREDP_VEC=0 ADC_SHAREDP_TMA=1 timeout 300 python tools/probe_shared_p.py 2>&1 | tail -2
done
