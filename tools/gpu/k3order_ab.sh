# A/B: K1 enqueued before K3 (default) vs K3 first (CITO_K3_FIRST=1); scp step and multistart
timeout 600 python -m pytest tests/test_scatter.py tests/test_subproblem.py -m gpu -x -q 2>&1 | tail -n 1
for e in "CITO_K3_FIRST=0" "CITO_K3_FIRST=1" "CITO_K3_FIRST=0" "CITO_K3_FIRST=1"; do
  env $e timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-fine-extra --no-batch-extra > gpurun_out/o_scp.json 2>/dev/null
  env $e timeout 600 python bench.py --workload multistart --steps 10 --no-cpu-baseline > gpurun_out/o_ms.json 2>/dev/null
  python -c "import json;a=json.load(open('gpurun_out/o_scp.json'));b=json.load(open('gpurun_out/o_ms.json'));print('$e', 'scp', round(a['ms_per_step'],4), 'e2e', round(a['e2e']['ms_per_step'],4), 'ms', round(b['ms_per_step'],4))"
done
