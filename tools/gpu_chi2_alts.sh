# Time alternative builds of the chi2 kernels (tools/alt_*.sed applied to
# chi2.cu / chi2_host.cpp in a scratch copy) against the tree's build,
# alternating runs.
O=gpurun_out; mkdir -p $O
for alt in tools/alt_*.sed; do
  name=$(basename $alt .sed)
  rm -rf /tmp/$name && mkdir /tmp/$name && cp -r paper_2203_06139_b200 include tools oracle /tmp/$name/
  (cd /tmp/$name && sed -i -f $alt paper_2203_06139_b200/csrc/chi2.cu paper_2203_06139_b200/csrc/chi2_host.cpp && make -s -j8 -C paper_2203_06139_b200/csrc > /tmp/${name}_build.log 2>&1) || echo "$name build failed"
done
for rep in 1 2; do
  echo "base: $(timeout 300 python tools/probe_chi2.py ${CHI2_BINS:-100000000} 20 2>&1 | tail -1)"
  for alt in tools/alt_*.sed; do
    name=$(basename $alt .sed)
    echo "$name: $(cd /tmp/$name && timeout 300 python tools/probe_chi2.py ${CHI2_BINS:-100000000} 20 2>&1 | tail -1)"
  done
done
