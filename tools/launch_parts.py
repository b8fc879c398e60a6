"""Host-side cost of the pieces of GpuSCPStep.iterate (microseconds; GPU box)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess
from paper_2604_09993_b200.subproblem import GpuSCPStep
sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)
step = GpuSCPStep(gt)
for _ in range(20): step.iterate(z, 1.0)
pl = step._plan; pat = step.asm.pat
def t(f, n=2000):
    for _ in range(50): f()
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
zp = pl["zde_pin"].numpy(); dim = pat.lay.dim
hb = step._host_buffer()
g = hb.graphs[False]
stream = torch.cuda.current_stream()
print("isfinite", t(lambda: np.all(np.isfinite(z))))
def fill():
    zp[:dim] = z; zp[dim] = 1.0; zp[dim + 1] = 1e-4
print("zp fill", t(fill))
print("host_buffer", t(lambda: step._host_buffer()))
print("objective_c", t(lambda: pat.objective_c(z)))
print("current_stream", t(lambda: torch.cuda.current_stream(gt.device)))
print("lazy lin", t(lambda: step._Lazy(hb.slot["lin"], z.copy())))
def rep():
    g.replay()
print("replay (+sync each 1)", t(lambda: (g.replay(), stream.synchronize()), 500))
print("sync idle", t(lambda: stream.synchronize()))
print("iterate total", t(lambda: step.iterate(z, 1.0), 500))
