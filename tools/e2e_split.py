"""Split GpuSCPStep.iterate wall time: launches / wait for the device / host post-processing.  (GPU box)

  python tools/e2e_split.py [--precondition] [--profile]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.subproblem import GpuSCPStep  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)
step = GpuSCPStep(gt)
pc = "--precondition" in sys.argv
for _ in range(20):
    step.iterate(z, 1.0, precondition=pc)
marks = []
orig_sync = torch.cuda.Stream.synchronize


def sync(self):
    marks.append(("before_sync", time.perf_counter()))
    orig_sync(self)
    marks.append(("after_sync", time.perf_counter()))


torch.cuda.Stream.synchronize = sync
tot = {"launch": [], "wait": [], "post": []}
for _ in range(200):
    marks.clear()
    t0 = time.perf_counter()
    step.iterate(z, 1.0, precondition=pc)
    t3 = time.perf_counter()
    t1 = [t for n, t in marks if n == "before_sync"][0]
    t2 = [t for n, t in marks if n == "after_sync"][0]
    tot["launch"].append(t1 - t0)
    tot["wait"].append(t2 - t1)
    tot["post"].append(t3 - t2)
print({k: round(float(np.median(v)) * 1e3, 4) for k, v in tot.items()}, "ms (median)")
print("packed D2H bytes", step._plan["pk"].nbytes, "copied per call", step.d2h_bytes(pc), "refetches",
      step.pattern_refetches)

if "--profile" in sys.argv:
    import cProfile
    import pstats

    torch.cuda.Stream.synchronize = orig_sync
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        step.iterate(z, 1.0, precondition=pc)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
