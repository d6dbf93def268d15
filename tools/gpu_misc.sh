mkdir -p gpurun_out
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for k in k_looped k_rational; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:adc_kernel_$k -s 2 -c 1 python tools/probe_jit.py $k > gpurun_out/ncu_fp64_$k.txt 2>&1
  grep -E "smsp__|sm__pipe|duration" gpurun_out/ncu_fp64_$k.txt
done
bash tools/gpu_sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1; cat gpurun_out/sanitize_summary.txt
