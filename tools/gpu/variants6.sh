timeout 600 python -m pytest tests/test_gpu_linearize.py tests/test_reference_models.py -m gpu -x -q 2>&1 | tail -1
for v in base "" base ""; do
  echo "variant=$v $(CITO_LIB_VARIANT=$v KNEE_B=29,29,199,4096 python tools/knee.py | tr '\n' ' ')"
done
