# A/B of the shared-mean form with dx: the tree against tools/_ab_gaussnd_base.cu
# (an alternative gaussnd.cu you place there), alternating runs.
rm -rf /tmp/ab && mkdir /tmp/ab && cp -r paper_2203_06139_b200 include tools oracle /tmp/ab/
cp tools/_ab_gaussnd_base.cu /tmp/ab/paper_2203_06139_b200/csrc/gaussnd.cu
(cd /tmp/ab && make -s -j8 -C paper_2203_06139_b200/csrc > /tmp/ab_build.log 2>&1) || echo "base build failed"
for rep in 1 2; do
  for cfg in "100 10000000" "37 27000000" "200 5000000"; do
    echo "tree [$cfg] $(python tools/probe_shared_p.py 5 $cfg | grep 'with dx' | cut -c1-40)"
    echo "base [$cfg] $(cd /tmp/ab && python tools/probe_shared_p.py 5 $cfg | grep 'with dx' | cut -c1-40)"
  done
done
