# round evidence refresh (v18): refresh.sh + ncu of the node kernel K3 at the multistart size
bash tools/gpu/refresh.sh
set -x
M="python bench.py --workload multistart --steps 3 --warmup 3 --no-cpu-baseline"
$M > gpurun_out/plain_ms.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_node -s 1 -c 1 -o gpurun_out/k3_ms $M > gpurun_out/ncu_k3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_ms.csv $M > gpurun_out/ncu_ms_launch.log 2>&1
ls gpurun_out
