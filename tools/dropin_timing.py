"""Per-call host timing of the module-level drop-ins (linearize_all, build_subproblem,
precondition) as the reference's SCP loop calls them.  (GPU box)"""
import sys
import time
from types import SimpleNamespace

import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, _cache, initial_guess  # noqa: E402
from paper_2604_09993_b200.scenario import build_scaling  # noqa: E402
from paper_2604_09993_b200.subproblem import build_subproblem, precondition  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)
tr = SimpleNamespace(scenario=sc, layout=gt.lay, scaling=SimpleNamespace(scale=build_scaling(sc, gt.lay)[0]))
_cache[id(tr)] = (tr, gt)
cfg = SimpleNamespace(w_prox=2000.0, w_ep=50000.0)
acc = {"linearize_all": 0.0, "build_subproblem": 0.0, "precondition": 0.0}
n = 50
for it in range(n + 5):
    t0 = time.perf_counter()
    lin = gt.linearize_all(z, 1.0)
    t1 = time.perf_counter()
    prog, meta = build_subproblem(tr, lin, z, 1.0, cfg)
    t2 = time.perf_counter()
    sc_prog, prec = precondition(prog)
    t3 = time.perf_counter()
    if it >= 5:
        acc["linearize_all"] += t1 - t0
        acc["build_subproblem"] += t2 - t1
        acc["precondition"] += t3 - t2
print({k: round(v / n * 1e3, 3) for k, v in acc.items()}, "ms per call")
