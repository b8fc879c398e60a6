"""Where does the e2e SCP step spend host time?  (GPU box)"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from types import SimpleNamespace
from paper_2604_09993_b200 import scenario as S
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess, _cache
from paper_2604_09993_b200.scenario import build_scaling
from paper_2604_09993_b200.subproblem import build_subproblem, _assemblers
import cProfile, pstats

sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)


class Tr:
    pass


tr = Tr()
tr.scenario, tr.layout = sc, gt.lay
tr.scaling = SimpleNamespace(scale=build_scaling(sc, gt.lay)[0])
_cache[id(tr)] = (tr, gt)
cfg = SimpleNamespace(w_prox=2000.0, w_ep=50000.0)
for _ in range(5):
    lin = gt.linearize_all(z, 1.0)
    prog, meta = build_subproblem(tr, lin, z, 1.0, cfg)
torch.cuda.synchronize()
n = 50
t0 = time.perf_counter()
for _ in range(n):
    lin = gt.linearize_all(z, 1.0)
    prog, meta = build_subproblem(tr, lin, z, 1.0, cfg)
print("e2e ms", (time.perf_counter() - t0) / n * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    lin = gt.linearize_all(z, 1.0)
    prog, meta = build_subproblem(tr, lin, z, 1.0, cfg)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
