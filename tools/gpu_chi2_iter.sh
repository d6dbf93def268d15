# chi2 kernel iteration on one B200: GPU parity suite, pass timing, ncu of
# the tile kernel, JIT timings, and (if tools/alt.sed exists) an alternative
# build of chi2.cu timed beside it.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; tail -4 $O/pytest_gpu.log
timeout 300 python tools/probe_chi2.py 100000000 20 > $O/probe_chi2.log 2>&1; tail -3 $O/probe_chi2.log
timeout 300 python tools/probe_fit_1e6.py > $O/probe_fit.log 2>&1; tail -3 $O/probe_fit.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chi2_tile -s 3 -c 1 -o $O/prof_chi2 python tools/probe_chi2.py 100000000 5 > $O/ncu_chi2.log 2>&1
python tools/ncu_summary.py $O/prof_chi2.ncu-rep > $O/ncu_summary.txt 2>&1
python tools/ncu_fp64_per_unit.py $O/prof_chi2.ncu-rep 1e8 >> $O/ncu_summary.txt 2>&1
timeout 600 python tools/probe_jit.py > $O/probe_jit.log 2>&1; tail -6 $O/probe_jit.log
for alt in tools/alt_*.sed; do
  [ -f "$alt" ] || continue
  name=$(basename $alt .sed)
  rm -rf /tmp/alt && mkdir /tmp/alt && cp -r paper_2203_06139_b200 include tools oracle /tmp/alt/ && cd /tmp/alt
  sed -i -f $alt paper_2203_06139_b200/csrc/chi2.cu paper_2203_06139_b200/csrc/chi2_host.cpp && make -s -j8 -C paper_2203_06139_b200/csrc > /tmp/alt_build.log 2>&1
  timeout 300 python tools/probe_chi2.py 100000000 20 > $GRAFT_REPO_ROOT/$O/probe_chi2_$name.log 2>&1; echo "$name: $(tail -1 $GRAFT_REPO_ROOT/$O/probe_chi2_$name.log)"
  cd $GRAFT_REPO_ROOT
done
