# K1 A/B check: parity tests (default K1 = v2), role timing and quick device timings of both versions
set -x
CITO_K1=2 timeout 600 python -m pytest tests/test_gpu_linearize.py tests/test_reference_models.py tests/test_subproblem.py -x -q -m gpu > gpurun_out/k1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1_pytest.log
CITO_K1=2 timeout 300 python tools/role_timing.py run 29 > gpurun_out/role29_v2.txt 2>&1
CITO_K1=2 timeout 300 python tools/role_timing.py run 4096 > gpurun_out/role4096_v2.txt 2>&1
CITO_K1=1 timeout 300 python tools/role_timing.py run 29 > gpurun_out/role29_v1.txt 2>&1
for v in 2 1; do CITO_K1=$v timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-fine-extra > gpurun_out/bench_k1v$v.json 2> gpurun_out/bench_k1v$v.err; done
tail -3 gpurun_out/k1_pytest.log; tail -4 gpurun_out/role29_v2.txt gpurun_out/role4096_v2.txt gpurun_out/role29_v1.txt
python - <<'PY'
import json
for v in (2, 1):
    try:
        d = json.load(open(f"gpurun_out/bench_k1v{v}.json"))
        print(v, d["ms_per_step"], d["roofline"]["kernel_ms"], d["batch_extra"]["ms_per_step"], d["e2e"]["ms_per_step"])
    except Exception as e:
        print(v, "fail", e)
PY
