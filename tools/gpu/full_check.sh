set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_scp.json 2> gpurun_out/bench_scp.err
timeout 600 python bench.py --workload batch --steps 20 > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
timeout 600 python bench.py --workload multistart --steps 10 --no-cpu-baseline > gpurun_out/bench_ms.json 2> gpurun_out/bench_ms.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cat gpurun_out/bench_*.json
