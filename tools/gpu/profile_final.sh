# ncu of the default kernels: latency K1 (29 intervals) and batch K1 (4096, 3 intervals/CTA)
set -x
python tools/prof_small.py 29 lin > gpurun_out/plain29.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1_scp python tools/prof_small.py 29 lin > gpurun_out/ncu_scp.log 2>&1
python tools/prof_small.py 4096 lin > gpurun_out/plain4096.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1_batch python tools/prof_small.py 4096 lin > gpurun_out/ncu_batch.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-batch-extra --no-fine-extra"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_scp.csv $B > gpurun_out/ncu_launch.log 2>&1
