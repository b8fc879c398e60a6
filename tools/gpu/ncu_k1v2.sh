set -x
CITO_K1=2 python tools/prof_small.py 29 > gpurun_out/plain.log 2>&1 && \
CITO_K1=2 ncu --set full --clock-control none --import-source on -k regex:k_linearize2 -s 2 -c 1 -o gpurun_out/k1v2b_29 python tools/prof_small.py 29 > gpurun_out/ncu1.log 2>&1
