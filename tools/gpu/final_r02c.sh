# round-2 closing bench lines after the host-side pre-build (one box, back to back)
set -x
O=gpurun_out/fin2
mkdir -p $O
python bench.py --steps 30 --warmup 5 > $O/bench_scp.json 2> $O/bench_scp.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --workload batch --steps 10 --warmup 3 > $O/bench_batch.json 2> $O/bench_batch.err
python bench.py --workload multistart --steps 5 --warmup 3 > $O/bench_ms.json 2> $O/bench_ms.err
python bench.py --workload fine --steps 20 --warmup 5 > $O/bench_fine.json 2> $O/bench_fine.err
{ python tools/e2e_split.py; python tools/e2e_split.py --precondition; } > $O/e2e_split.txt 2>&1
python tools/scp_solve_profile.py 8 30 --one-pass --idle-probe > $O/solve_install_scp.json 2> $O/solve_install_scp.err
python tools/models_timing.py > $O/models_timing.txt 2>&1
cp gpurun_out/models_timing.json $O/ 2>/dev/null
for f in $O/bench_*.err; do echo $f; tail -c 300 $f; done
