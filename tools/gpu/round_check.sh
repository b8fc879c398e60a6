# full GPU test suite (both K1 generations for the linearize parity tests), smoke, default bench
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
CITO_K1=2 timeout 600 python -m pytest tests/test_gpu_linearize.py tests/test_reference_models.py tests/test_subproblem.py -m gpu -x -q > gpurun_out/pytest_gpu_k1v2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_k1v2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_scp.json 2> gpurun_out/bench_scp.err
timeout 600 python bench.py --workload fine --steps 10 --no-cpu-baseline > gpurun_out/bench_fine.json 2> gpurun_out/bench_fine.err
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/pytest_gpu_k1v2.log gpurun_out/smoke.log
cat gpurun_out/bench_scp.json gpurun_out/bench_fine.json
