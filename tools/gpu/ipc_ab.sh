CITO_K1_IPC3=1 timeout 600 python -m pytest tests/test_gpu_linearize.py -q -m gpu -x 2>&1 | tail -1
for e in "" "CITO_K1_IPC3=1" "" "CITO_K1_IPC3=1"; do
  env $e timeout 600 python bench.py --workload batch --steps 10 --no-cpu-baseline > gpurun_out/ipc.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ipc.json'));print('$e', d['ms_per_step'], d['roofline']['frac'])"
done
