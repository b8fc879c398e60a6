"""K3 generations agree bit for bit: the warp-per-item kernel (k_node_w, default;
live directions only, structural columns written as zero / identity) against the
thread-per-(item, direction) kernel (k_node, CITO_K3=1) on every golden model and a
HalfCheetah multi-start batch.  Runs each generation in its own process (the
switch is read once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
from conftest import golden_scenario, load_golden
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess_batch
res = {}
for name in ("pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"):
    g = load_golden(name)
    gt = GpuTranscription(golden_scenario(name))
    for tag, z in (("ig", g["ig_z"]), ("nd", g["nd_z"])):
        r = gt.linearize_device(torch.as_tensor(z, device=gt.device), 0.05)
        for k in ("psi", "psi_jac", "theta", "theta_jac", "imp_v", "imp_jac"):
            res[f"{name}_{tag}_{k}"] = r[k].cpu().numpy()
sc = golden_scenario("halfcheetah_n30")
gt = GpuTranscription(sc)
Z = initial_guess_batch(sc, gt.disc, list(range(6)), gt.lay)
r = gt.linearize_device(torch.as_tensor(Z, device=gt.device), 1.0)
for k in ("psi", "psi_jac", "theta", "theta_jac", "imp_v", "imp_jac"):
    res[f"ms_{k}"] = r[k].cpu().numpy()
np.savez(OUT, **res)
"""


def _run(tmp, k3):
    out = os.path.join(tmp, f"k3_{k3}.npz")
    env = dict(os.environ)
    env.pop("CITO_K3", None)
    if k3:
        env["CITO_K3"] = k3
    code = f"ROOT = {ROOT!r}\nOUT = {out!r}\n" + SCRIPT
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return dict(np.load(out))


@pytest.mark.gpu
def test_node_kernel_generations_bit_identical(tmp_path):
    a = _run(str(tmp_path), "")
    b = _run(str(tmp_path), "1")
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_live_direction_tables():
    """The live-direction rule of k_node_w (NodeDirs in csrc/cito_node.cuh) restated:
    HalfCheetah (flat) impulse map 32 of 67, theta 24 of 69."""
    nq, nc = 21, 2
    contact_links = (3, 6)
    imp = [d for d in range(3 * nq + 2 * nc)
           if (d < nq and d % 3 == 2) or (nq <= d < 2 * nq) or d >= 3 * nq]
    th = [d for d in range(3 * nq + 3 * nc) if (d >= 3 * nq) or ((d % nq) // 3 in contact_links)]
    assert len(imp) == 32 and len(th) == 24
