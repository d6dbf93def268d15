for m in 8 4 3 2 1; do echo -n "margin $m: "; ADC_FIT_MARGIN=$m timeout 300 python tools/probe_fit_launches.py 400; done
