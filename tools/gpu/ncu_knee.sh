set -x
for B in 29 148; do
python tools/prof_small.py $B lin > gpurun_out/plain_$B.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_linearize -s 2 -c 1 -o gpurun_out/knee_$B python tools/prof_small.py $B lin > gpurun_out/ncu_knee_$B.log 2>&1
done
