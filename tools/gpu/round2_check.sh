python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py --steps 20 --warmup 5 > gpurun_out/b3.json 2> gpurun_out/b3.err; tail -c 400 gpurun_out/b3.err
CITO_CSC_RECIPES=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-batch-extra --no-fine-extra > gpurun_out/b3_recipes.json 2>> gpurun_out/b3.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_b3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-batch-extra --no-fine-extra > gpurun_out/ncu_b3.log 2>&1
