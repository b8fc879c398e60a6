# round-2 bench lines for profiles/ (one box, back to back)
python bench.py --steps 30 --warmup 5 > gpurun_out/r02_bench_scp.json 2> gpurun_out/r02_bench_scp.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
python bench.py --workload batch --steps 10 --warmup 3 > gpurun_out/r02_bench_batch.json 2> gpurun_out/r02_bench_batch.err
python bench.py --workload multistart --steps 5 --warmup 3 > gpurun_out/r02_bench_ms.json 2> gpurun_out/r02_bench_ms.err
python bench.py --workload fine --steps 20 --warmup 5 > gpurun_out/r02_bench_fine.json 2> gpurun_out/r02_bench_fine.err
python tools/e2e_split.py > gpurun_out/r02_e2e_split.txt 2>&1
python tools/e2e_split.py --precondition >> gpurun_out/r02_e2e_split.txt 2>&1
python tools/scp_solve_profile.py 6 30 --one-pass > gpurun_out/r02_scp_onepass.json 2> gpurun_out/r02_scp_onepass.err
python tools/scp_solve_profile.py 6 30 > gpurun_out/r02_scp_three.json 2> gpurun_out/r02_scp_three.err
for f in gpurun_out/r02_bench_*.err; do echo $f; tail -c 300 $f; done
