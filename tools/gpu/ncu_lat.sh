python tools/prof_small.py 29 lin > gpurun_out/plain29.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1_lat python tools/prof_small.py 29 lin > gpurun_out/ncu_lat.log 2>&1
