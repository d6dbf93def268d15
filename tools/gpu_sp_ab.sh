# A/B of the shared-mean forms: the tree against tools/_ab_gaussnd_base.cu
# (+ tools/_ab_capi_base.cpp if present), alternatives you place there, built
# in a scratch copy; alternating runs.
rm -rf /tmp/ab && mkdir /tmp/ab && cp -r paper_2203_06139_b200 include tools oracle /tmp/ab/
cp tools/_ab_gaussnd_base.cu /tmp/ab/paper_2203_06139_b200/csrc/gaussnd.cu
[ -f tools/_ab_capi_base.cpp ] && cp tools/_ab_capi_base.cpp /tmp/ab/paper_2203_06139_b200/csrc/capi.cpp
(cd /tmp/ab && make -s -j8 -C paper_2203_06139_b200/csrc > /tmp/ab_build.log 2>&1) || echo "base build failed"
for rep in 1 2; do
  for cfg in ${AB_CFGS:-"100 10000000" "37 27000000" "200 5000000"}; do
    echo "tree [$cfg] $(python tools/probe_shared_p.py 5 $cfg | cut -c1-40 | tr '\n' '|')"
    echo "base [$cfg] $(cd /tmp/ab && python tools/probe_shared_p.py 5 $cfg | cut -c1-40 | tr '\n' '|')"
  done
  for d in 37 100; do
    echo "tree $(python tools/probe_shared_p_views.py $d 5000000 | grep 'odd view' | tr '\n' '|')"
    echo "base $(cd /tmp/ab && python tools/probe_shared_p_views.py $d 5000000 | grep 'odd view' | tr '\n' '|')"
  done
done
