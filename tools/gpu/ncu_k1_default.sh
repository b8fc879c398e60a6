set -x
python tools/prof_small.py 29 lin > gpurun_out/plain29.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1_scp python tools/prof_small.py 29 lin > gpurun_out/ncu_scp.log 2>&1
python tools/prof_small.py 29 prop > gpurun_out/plain29p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k2_prop python tools/prof_small.py 29 prop > gpurun_out/ncu_prop.log 2>&1
