"""Host-side breakdown of GpuSCPStep.iterate (the bench's e2e call).  (GPU box)"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.subproblem import GpuSCPStep  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)
step = GpuSCPStep(gt)
for pc in (False, True):
    for _ in range(10):
        step.iterate(z, 1.0, precondition=pc)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        step.iterate(z, 1.0, precondition=pc)
    print("precondition", pc, "e2e ms", (time.perf_counter() - t0) / n * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    step.iterate(z, 1.0)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
