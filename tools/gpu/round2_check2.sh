python -m pytest tests -m gpu -q -x -k "reference_models or reference_integration" 2>&1 | tail -15
python tools/scp_solve_profile.py 6 30 --one-pass > gpurun_out/scp_onepass.json 2> gpurun_out/scp_onepass.err
python tools/scp_solve_profile.py 6 30 > gpurun_out/scp_three.json 2> gpurun_out/scp_three.err
tail -c 500 gpurun_out/scp_onepass.err
