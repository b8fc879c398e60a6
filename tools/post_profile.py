"""cProfile of GpuSCPStep.iterate's host side (GPU box)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.subproblem import GpuSCPStep  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)
step = GpuSCPStep(gt)
for _ in range(20):
    step.iterate(z, 1.0)
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    step.iterate(z, 1.0)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
