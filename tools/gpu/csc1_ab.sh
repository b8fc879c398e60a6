# one-pass CSC compaction: subproblem/precondition parity + scp step A/B vs the two-launch version (CITO_CSC2=1)
timeout 600 python -m pytest tests/test_subproblem.py tests/test_precondition.py tests/test_reference_integration.py -q -m gpu -x 2>&1 | tail -n 2
CITO_CSC2=1 timeout 600 python -m pytest tests/test_subproblem.py -q -m gpu -x 2>&1 | tail -n 1
for e in "" "CITO_CSC2=1" "" "CITO_CSC2=1"; do
  env $e timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-fine-extra --no-batch-extra > gpurun_out/csc.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/csc.json'));print('$e', d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'], d['gpu_launches'])"
done
