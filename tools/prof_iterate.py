"""GpuSCPStep.iterate of HalfCheetah N=30 with eager launches (for ncu captures of the
kernels of one SCP iteration as the public API runs them).  (GPU box)

  python tools/prof_iterate.py [calls] [--precondition]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.subproblem import GpuSCPStep  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 5
sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)
step = GpuSCPStep(gt, use_graph=False)
for _ in range(calls):
    step.iterate(z, 1.0, precondition="--precondition" in sys.argv)
torch.cuda.synchronize()
print("ok", calls, "calls; d2h bytes", step.d2h_copied)
