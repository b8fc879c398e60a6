"""Exact-zero pattern of the GPU node Jacobians vs the reference goldens (diagnostic)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from conftest import load_golden, golden_scenario  # noqa
from paper_2604_09993_b200.linearize import GpuTranscription

for name in ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]:
    g = load_golden(name)
    gt = GpuTranscription(golden_scenario(name))
    lin = gt.linearize_all(g["ig_z"], float(g["ig_delta"]))
    for f, k in (("psi_jac", "ig_psi_jac"), ("theta_jac", "ig_theta_jac"), ("imp_jac", "ig_imp_jac"), ("jx", "ig_jx"), ("ju", "ig_ju")):
        a, b = getattr(lin, f), g[k]
        za, zb = a == 0, b == 0
        bad = np.argwhere(za != zb)
        print(name, f, "pattern mismatches", len(bad), "max abs diff", np.abs(a - b).max())
        for idx in bad[:6]:
            print("   ", tuple(idx), a[tuple(idx)], b[tuple(idx)])
