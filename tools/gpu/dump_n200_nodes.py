"""Dump the GPU linearize_all outputs at the configs[4] golden point (N=200, 8
substeps) into gpurun_out/ for an offline zero-pattern comparison."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden_scenario, load_golden  # noqa: E402

from paper_2604_09993_b200.linearize import GpuTranscription  # noqa: E402

g = load_golden("halfcheetah_n200s8")
gt = GpuTranscription(golden_scenario("halfcheetah_n200s8"))
r = gt.linearize_device(torch.as_tensor(g["ig_z"], device=gt.device), 1.0)
torch.cuda.synchronize()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "n200_gpu.npz"), **{k: v.cpu().numpy() for k, v in r.items()})
for k in ("jx", "ju", "js", "psi_jac", "theta_jac", "imp_jac"):
    a, b = r[k].cpu().numpy(), g["ig_" + k]
    d = (a == 0) != (b == 0)
    print(k, "pattern diffs", int(d.sum()), "at", np.argwhere(d)[:8].tolist())
