"""bench.py's record contract on the host side (no GPU): both arms describe the
workload with the same `config` dict (the driver compares them), the metric is
BASELINE.json's, and --gpus N without torchrun re-launches under torch.distributed.run."""
import json
import os
import sys
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(**kw):
    a = dict(workload="scp", batch=4096, problems=1024)
    a.update(kw)
    return SimpleNamespace(**a)


def test_metric_is_baselines():
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert bench.METRIC == base["metric"]


def test_config_identical_for_both_arms_and_free_of_model_keys():
    for wl in ("scp", "fine", "batch", "multistart"):
        for world in (1, 2, 8):
            c1 = bench.config_for(_args(workload=wl), world)
            c2 = bench.config_for(_args(workload=wl), world)
            assert c1 == c2 and "workload" in c1 and "model" not in c1
            if wl in ("scp", "fine"):
                assert c1["parallelism"].startswith("replicas")
            else:
                assert c1["parallelism"].startswith("shards" if world > 1 else "single GPU")


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, cwd=None: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    try:
        bench.relaunch_under_torchrun(SimpleNamespace(gpus=4))
    except SystemExit as e:
        assert e.code == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
