# default K1: parity tests, per-role cycle timing, short bench (scp + batch extra)
set -x
timeout 600 python -m pytest tests/test_gpu_linearize.py tests/test_reference_models.py tests/test_subproblem.py tests/test_verifier.py -x -q -m gpu > gpurun_out/k1q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1q_pytest.log
timeout 300 python tools/role_timing.py run 29 > gpurun_out/role29.txt 2>&1
timeout 300 python tools/role_timing.py run 4096 > gpurun_out/role4096.txt 2>&1
timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-fine-extra > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -n 3 gpurun_out/k1q_pytest.log
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_q.json"))
print("step", d["ms_per_step"], "k1", d["roofline"]["kernel_ms"], "batch", d["batch_extra"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"])
PY
