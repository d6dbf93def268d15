# compute-sanitizer over the product kernels (small parity cases): memcheck
# (out-of-bounds / misaligned global and shared accesses), racecheck (shared
# memory hazards), synccheck, initcheck; and the C++ mirror's check program
# (incl. 4 host threads on distinct buffers) under memcheck and racecheck.
# Logs -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
# torch must not pool allocations, or memcheck only sees its 2 MB segments
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
SEL="claimed_spans_match or claimed_spans_in_cuda_graph or shared_p_with_dx or golden or listing1_cases or domain_error or shared_p_golden or multi_bitwise or numeric_provider_probe or accumulates_twice or sample_histogram_zero or compute_shared_forced or chi2_gradient_batch or corpus_gradient or high_counts"
# racecheck / synccheck cannot follow the fit's device-side loop (a CUDA graph
# WHILE node): they run the kernels without the device-loop fits (the fits'
# kernels are the same chi2 / multi kernels the other cases launch)
NOFIT="and not fit and not sample_histogram_zero and not high_counts"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  sel="${SELECT:-$SEL}"
  case $tool in racecheck|synccheck) sel="($sel) $NOFIT";; esac
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 0 --print-limit 50 \
    --log-file gpurun_out/sanitize_${tool}.log \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_jit.py -q -x -m gpu -k "$sel" -p no:cacheprovider \
    > gpurun_out/sanitize_${tool}_pytest.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitize_${tool}_pytest.log)"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|Uninitialized" gpurun_out/sanitize_${tool}.log | sort | uniq -c | head -8
done
# the fit's kernels through the host loop
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 0 --log-file gpurun_out/sanitize_fit_${tool}.log \
    python tools/sanitize_fit_hostloop.py > gpurun_out/sanitize_fit_${tool}_out.log 2>&1
  echo "fit (host loop) $tool rc=$? $(tail -1 gpurun_out/sanitize_fit_${tool}_out.log) | $(grep -E 'SUMMARY' gpurun_out/sanitize_fit_${tool}.log | sort | uniq -c)"
done
# the C++ mirror check (error contract, 4 threads on distinct buffers, the
# multi-GPU host form) under memcheck and racecheck
make -s -C oracle restate
g++ -std=c++17 -O2 -Wall -I include -I oracle tests/cpu/cxx_api_check.cpp oracle/restate.c -x none \
    -L paper_2203_06139_b200 -ladc_b200 -Wl,-rpath,$PWD/paper_2203_06139_b200 -o /tmp/cxx_api_check -lpthread
for tool in memcheck racecheck synccheck; do
  mode=gpu; [ $tool = memcheck ] || mode=gpu-launch
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 0 --log-file gpurun_out/sanitize_cxx_${tool}.log \
    /tmp/cxx_api_check $mode > gpurun_out/sanitize_cxx_${tool}_out.log 2>&1
  echo "cxx $tool rc=$? $(tail -1 gpurun_out/sanitize_cxx_${tool}_out.log) | $(grep 'ERROR SUMMARY' gpurun_out/sanitize_cxx_${tool}.log | sort | uniq -c)"
done
# canary: an out-of-bounds launch must be reported (the tool is attached)
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/sanitize_canary.py > gpurun_out/sanitize_canary.log 2>&1
echo "canary: $(grep -c 'Invalid __global__' gpurun_out/sanitize_canary.log) invalid-access reports; $(grep 'ERROR SUMMARY' gpurun_out/sanitize_canary.log)"
