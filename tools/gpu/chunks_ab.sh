# chunked D2H pipeline of cito_linearize_host: tests + batch e2e A/B (CITO_HOST_CHUNKS=0 = one launch, copies after)
timeout 600 python -m pytest tests/test_gpu_linearize.py -m gpu -x -q 2>&1 | tail -n 3
for e in "CITO_HOST_CHUNKS=1" "CITO_HOST_CHUNKS=0" "CITO_HOST_CHUNKS=1" "CITO_HOST_CHUNKS=0"; do
  env $e timeout 600 python bench.py --workload batch --steps 20 --no-cpu-baseline > gpurun_out/c_b.json 2>gpurun_out/c_b.err
  python -c "import json;b=json.load(open('gpurun_out/c_b.json'));print('$e', 'ms', round(b['ms_per_step'],4), 'e2e', round(b['e2e']['ms_per_step'],4), b['e2e']['value'])" || tail -5 gpurun_out/c_b.err
done
