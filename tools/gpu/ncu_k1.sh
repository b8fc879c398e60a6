# ncu --set full of the K1 kernel (v2 and v1) on the 29-interval latency case
set -x
python tools/prof_small.py 29 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_linearize2 -s 2 -c 1 -o gpurun_out/k1v2_29 python tools/prof_small.py 29 > gpurun_out/ncu1.log 2>&1
CITO_K1=1 python tools/prof_small.py 29 > gpurun_out/plain1.log 2>&1 && \
CITO_K1=1 ncu --set full --clock-control none --import-source on -k regex:k_linearize -s 2 -c 1 -o gpurun_out/k1v1_29 python tools/prof_small.py 29 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
