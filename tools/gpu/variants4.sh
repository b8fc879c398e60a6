for v in base "" base ""; do
  echo "== variant=$v"
  CITO_LIB_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_linearize.py -q -m gpu -x 2>&1 | tail -1
  CITO_LIB_VARIANT=$v KNEE_B=29,199 python tools/knee.py | tr '\n' ' '; echo
  CITO_LIB_VARIANT=$v timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-fine-extra > gpurun_out/bb_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bb_$v.json'));print('scp', d['ms_per_step'], d['roofline']['kernel_ms'], 'batch', d['batch_extra']['ms_per_step'])"
done
