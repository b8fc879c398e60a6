# K3 (node kernel) change: full GPU parity suite, multistart bench, K3/K1 launch times (ncu launch list)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/nc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/nc_pytest.log
timeout 600 python bench.py --workload multistart --steps 10 --no-cpu-baseline > gpurun_out/nc_ms.json 2> gpurun_out/nc_ms.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_node --csv --log-file gpurun_out/nc_launches.csv python bench.py --workload multistart --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -n 2 gpurun_out/nc_pytest.log
python -c "import json;d=json.load(open('gpurun_out/nc_ms.json'));print('ms', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
grep -o '"ns","[0-9.]*"' gpurun_out/nc_launches.csv | tail -3
