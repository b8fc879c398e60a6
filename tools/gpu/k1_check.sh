python tools/role_timing.py run 29 > gpurun_out/role29.txt 2>&1
python -m pytest tests -m gpu -q -x -k "linearize or reference_models or fine_grid or subproblem" 2>&1 | tail -4
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fine-extra > gpurun_out/bk1.json 2> gpurun_out/bk1.err; tail -c 300 gpurun_out/bk1.err
