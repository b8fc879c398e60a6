# A/B of library variants on the default bench (scp + batch extra); parity for each
for v in "" split "" split; do
  CITO_LIB_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_linearize.py -q -m gpu -x 2>&1 | tail -1
  CITO_LIB_VARIANT=$v timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-fine-extra --no-batch-extra > gpurun_out/bv_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bv_$v.json'));print('variant=$v', d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step'])"
done
