rm -rf /tmp/ab && mkdir /tmp/ab && cp -r paper_2203_06139_b200 include tools oracle /tmp/ab/
cp tools/_ab_gaussnd_base.cu /tmp/ab/paper_2203_06139_b200/csrc/gaussnd.cu
(cd /tmp/ab && make -s -j8 -C paper_2203_06139_b200/csrc > /tmp/ab_build.log 2>&1) || echo "base build failed"
for rep in 1 2; do
  for d in 37 100 200; do
    echo "tree $(python tools/probe_shared_p_views.py $d 5000000 | grep 'odd view with dx')"
    echo "base $(cd /tmp/ab && python tools/probe_shared_p_views.py $d 5000000 | grep 'odd view with dx')"
  done
done
timeout 600 python -m pytest tests -q -m gpu -x -k "shared_p or multirank" 2>&1 | tail -1
