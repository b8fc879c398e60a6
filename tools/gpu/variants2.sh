for v in "" loop; do
  echo "== variant=$v"
  CITO_LIB_VARIANT=$v CITO_K1=1 timeout 300 python -m pytest tests/test_gpu_linearize.py -q -m gpu -x 2>&1 | tail -1
  CITO_LIB_VARIANT=$v CITO_K1=1 python tools/knee.py
  CITO_LIB_VARIANT=$v timeout 600 python bench.py --workload batch --steps 10 --no-cpu-baseline > gpurun_out/bb_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bb_$v.json'));print('batch', d['ms_per_step'], d['roofline']['frac'])"
done
