# bench.py's multi-rank paths with 2 ranks on ONE GPU over gloo (code-path check only:
# no kernel waits on another rank; timings are not multi-GPU numbers)
export CITO_BENCH_BACKEND=gloo CITO_BENCH_DEVICE=0
for w in scp batch multistart; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 3 --warmup 3 --workload $w --problems 64 --no-fine-extra > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "$w rc=$?"; tail -c 300 gpurun_out/mr_$w.err
done
python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 --workload batch > gpurun_out/ref_batch.json 2>&1; echo ref rc=$?
