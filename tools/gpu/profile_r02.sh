# round-2 evidence for profiles/: launch list of the bench step, full ncu captures of
# K1 (latency + batch), K3 (multistart), the entry-parallel CSC compaction, and the
# executed fp64 instruction counts of K1.  Every ncu run follows a plain run of the
# same command that exited 0.
set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-batch-extra --no-fine-extra"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_scp.csv $B > gpurun_out/ncu_launch.log 2>&1
python tools/prof_small.py 29 lin > gpurun_out/plain29.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1_scp python tools/prof_small.py 29 lin > gpurun_out/ncu_scp.log 2>&1
python tools/prof_small.py 4096 lin > gpurun_out/plain4096.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1_batch python tools/prof_small.py 4096 lin > gpurun_out/ncu_batch.log 2>&1
python tools/k3_time.py > gpurun_out/plain_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_node -s 2 -c 1 -o gpurun_out/k3_ms python tools/k3_time.py > gpurun_out/ncu_k3.log 2>&1
python tools/step_time.py 30 > gpurun_out/plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_csc_flat -s 2 -c 1 -o gpurun_out/csc_flat python tools/step_time.py 30 > gpurun_out/ncu_csc.log 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
for n in 29 4096; do
python tools/prof_small.py $n lin > gpurun_out/plain_$n.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:k_linearize -s 2 -c 1 --csv --log-file gpurun_out/fp64count_$n.csv python tools/prof_small.py $n lin > gpurun_out/ncu_fp64_$n.log 2>&1
done

# summaries on the box (the reports are too large to bring back together)
for r in k1_scp k1_batch k3_ms csc_flat; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_source.csv 2>/dev/null
  gzip -f gpurun_out/${r}_source.csv
done
rm -f gpurun_out/*.ncu-rep

ls -la gpurun_out
