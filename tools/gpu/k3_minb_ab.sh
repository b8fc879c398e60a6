# A/B of the K3 register cap (launch-bounds min blocks): default vs 6 vs 8 blocks/SM
timeout 600 python -m pytest tests/test_scatter.py -m gpu -x -q 2>&1 | tail -n 1
for v in "" k3m6 k3m8 "" k3m6 k3m8; do
  CITO_LIB_VARIANT=$v timeout 600 python bench.py --workload multistart --steps 10 --no-cpu-baseline > gpurun_out/v_ms.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/v_ms.json'));print('variant=$v', 'ms', round(b['ms_per_step'],4))"
done
for v in "" k3m6 k3m8; do
  CITO_LIB_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_node --csv --log-file gpurun_out/k3v_$v.csv python bench.py --workload multistart --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "variant=$v"; grep -o '"ns","[0-9.]*"' gpurun_out/k3v_$v.csv | tail -2
done
CITO_LIB_VARIANT=k3m8 timeout 600 python -m pytest tests/test_scatter.py tests/test_subproblem.py -m gpu -x -q 2>&1 | tail -n 1
