# round evidence refresh: full GPU tests, smoke, bench lines (all workloads), reference arm, ncu of the default K1s
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_scp.json 2> gpurun_out/bench_scp.err
timeout 600 python bench.py --workload batch --steps 20 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
timeout 600 python bench.py --workload multistart --steps 10 --no-cpu-baseline > gpurun_out/bench_ms.json 2> gpurun_out/bench_ms.err
timeout 600 python bench.py --workload fine --steps 10 > gpurun_out/bench_fine.json 2> gpurun_out/bench_fine.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/prof_small.py 29 lin > gpurun_out/plain29.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1_scp python tools/prof_small.py 29 lin > gpurun_out/ncu_scp.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-batch-extra --no-fine-extra"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_scp.csv $B > gpurun_out/ncu_launch.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
