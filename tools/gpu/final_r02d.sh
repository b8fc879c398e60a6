# round-2 closing evidence, final build (one box, back to back): bench lines of every
# workload + the reference arm, e2e split, graph timelines, the reference's solve loop
# with install_scp, models timing, role timing, then the ncu launch list and full
# captures of K1 (latency, batch) and the compaction, executed fp64 counts.
set -x
O=gpurun_out/fin3
mkdir -p $O
python bench.py --steps 30 --warmup 5 > $O/bench_scp.json 2> $O/bench_scp.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --workload batch --steps 10 --warmup 3 > $O/bench_batch.json 2> $O/bench_batch.err
python bench.py --workload multistart --steps 5 --warmup 3 > $O/bench_ms.json 2> $O/bench_ms.err
python bench.py --workload fine --steps 20 --warmup 5 > $O/bench_fine.json 2> $O/bench_fine.err
{ python tools/e2e_split.py; python tools/e2e_split.py --precondition; } > $O/e2e_split.txt 2>&1
{ python tools/graph_timeline.py; python tools/graph_timeline.py --precondition; python tools/graph_timeline.py --fine; } > $O/graph_timeline.txt 2>/dev/null
python tools/scp_solve_profile.py 8 30 --one-pass --idle-probe > $O/solve_install_scp.json 2> $O/solve_install_scp.err
python tools/models_timing.py > $O/models_timing.txt 2>&1
python tools/role_timing.py run 29 > $O/role_timing.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-batch-extra --no-fine-extra"
$B > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_scp.csv $B > $O/ncu_launch.log 2>&1
python tools/prof_small.py 29 lin > $O/plain29.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o $O/k1_scp python tools/prof_small.py 29 lin > $O/ncu_scp.log 2>&1
python tools/prof_small.py 4096 lin > $O/plain4096.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o $O/k1_batch python tools/prof_small.py 4096 lin > $O/ncu_batch.log 2>&1
python tools/prof_iterate.py 5 > $O/plain_iter.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_csc_flat -s 2 -c 1 -o $O/csc_flat python tools/prof_iterate.py 5 > $O/ncu_csc.log 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
for n in 29 4096; do
python tools/prof_small.py $n lin > $O/plain_$n.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:k_linearize -s 2 -c 1 --csv --log-file $O/fp64count_$n.csv python tools/prof_small.py $n lin > $O/ncu_fp64_$n.log 2>&1
done
for r in k1_scp k1_batch csc_flat; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page source --csv --print-source sass > $O/${r}_source.csv 2>/dev/null
  gzip -f $O/${r}_source.csv
done
rm -f $O/*.ncu-rep
ls -la $O | wc -l
