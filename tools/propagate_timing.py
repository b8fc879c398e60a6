"""Device time of Discretizer.propagate_batch_device for small and large batches.  (GPU box)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import Discretizer, scenario as S, synth  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
g, n_g = sc.path_constraints()
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
dev = torch.device("cuda")
for B in (1, 29, 148, 4096):
    x, U, Sv = synth.random_intervals(sc, B, seed=0)
    xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
    for _ in range(3):
        disc.propagate_batch_device(xd, Ud, Sd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 20
    for _ in range(n):
        disc.propagate_batch_device(xd, Ud, Sd)
    e1.record()
    torch.cuda.synchronize()
    print(f"propagate B={B}: {e0.elapsed_time(e1) / n * 1e3:.1f} us per call")
