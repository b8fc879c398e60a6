# executed fp64 thread-instructions of K1 (latency: 29 intervals; batch: 4096) for the flop-count cross-check
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
for B in 29 4096; do
python tools/prof_small.py $B lin > gpurun_out/plain_$B.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:k_linearize -s 2 -c 1 --csv --log-file gpurun_out/fp64count_$B.csv python tools/prof_small.py $B lin > gpurun_out/ncu_fp64_$B.log 2>&1
done
