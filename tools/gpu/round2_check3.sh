python -m pytest tests -m gpu -q -x -k "reference_integration or subproblem or fine_grid or precondition" 2>&1 | tail -5
python tools/scp_solve_profile.py 6 30 --one-pass > gpurun_out/scp_onepass.json 2> gpurun_out/scp_onepass.err
tail -c 500 gpurun_out/scp_onepass.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-batch-extra --no-fine-extra > gpurun_out/b4.json 2> gpurun_out/b4.err
