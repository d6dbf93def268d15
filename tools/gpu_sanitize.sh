# compute-sanitizer over the product kernels (small parity cases): memcheck
# (out-of-bounds / misaligned global and shared accesses), racecheck (shared
# memory hazards), synccheck, initcheck.  Logs -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
# torch must not pool allocations, or memcheck only sees its 2 MB segments
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
SEL="golden or listing1_cases or domain_error or shared_p_golden or multi_bitwise or numeric_provider_probe or accumulates_twice or sample_histogram_zero or compute_shared_forced"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  true
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 0 --print-limit 50 \
    --log-file gpurun_out/sanitize_${tool}.log \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_jit.py -q -x -m gpu -k "${SELECT:-$SEL}" -p no:cacheprovider \
    > gpurun_out/sanitize_${tool}_pytest.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitize_${tool}_pytest.log)"
  grep -E "ERROR SUMMARY|Invalid|Race|Uninitialized" gpurun_out/sanitize_${tool}.log | sort | uniq -c | head -8
done
# canary: an out-of-bounds launch must be reported (the tool is attached)
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/sanitize_canary.py > gpurun_out/sanitize_canary.log 2>&1
echo "canary: $(grep -c 'Invalid __global__' gpurun_out/sanitize_canary.log) invalid-access reports; $(grep 'ERROR SUMMARY' gpurun_out/sanitize_canary.log)"
