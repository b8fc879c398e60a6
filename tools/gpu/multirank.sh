# multi-rank bench code path on ONE GPU (gloo, 2 ranks on cuda:0; host-side collectives only)
export CITO_BENCH_BACKEND=gloo CITO_BENCH_DEVICE=0
for w in scp multistart; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --steps 5 --warmup 3 --workload $w --problems 16 > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "$w rc=$?"; tail -c 400 gpurun_out/mr_$w.json; echo
done
