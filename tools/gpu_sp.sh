for dn in "150 6666666" "200 5000000" "300 3333334" "500 2000000"; do
  for cfg in "8 2" "4 4" "4 3" "2 8" "2 6"; do
    set -- $cfg
    echo -n "dim/n $dn W=$1 cps=$2: "; ADC_GAUSSND_W=$1 ADC_GAUSSND_CPS=$2 timeout 120 python tools/probe_gaussnd_variants.py $dn 0 | grep variant
  done
done
