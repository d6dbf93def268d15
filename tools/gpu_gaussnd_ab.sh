# A/B: the tree's gaussnd.cu against tools/_ab_gaussnd_base.cu (a copy of an
# alternative you place there; built in a scratch copy), alternating probe runs.
rm -rf /tmp/ab && mkdir /tmp/ab && cp -r paper_2203_06139_b200 include tools oracle /tmp/ab/
cp tools/_ab_gaussnd_base.cu /tmp/ab/paper_2203_06139_b200/csrc/gaussnd.cu
(cd /tmp/ab && make -s -j8 -C paper_2203_06139_b200/csrc > /tmp/ab_build.log 2>&1) || echo "base build failed"
for rep in 1 2 3; do
  for cfg in ${AB_CFGS:-"1000 1000000" "1000 1000003" "200 5000001"}; do
    echo "tree [$cfg] $(python tools/probe_gaussnd_variants.py $cfg 0 | tail -1)"
    echo "base [$cfg] $(cd /tmp/ab && python tools/probe_gaussnd_variants.py $cfg 0 | tail -1)"
  done
done
