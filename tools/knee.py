import sys, torch
sys.path.insert(0, ".")
from paper_2604_09993_b200 import Discretizer, scenario as S, synth
sc = S.bundled("halfcheetah_bound", N=30)
g, n_g = sc.path_constraints()
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
dev = torch.device("cuda")
import os
BS = [int(x) for x in os.environ.get('KNEE_B', '29,60,74,75,96,120,140,148,149,199').split(',')]
for B in BS:
    x, U, Sv = synth.random_intervals(sc, B, seed=0)
    xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
    out = disc.linearize_batch_device(xd, Ud, Sd)
    for _ in range(3): disc.linearize_batch_device(xd, Ud, Sd, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): disc.linearize_batch_device(xd, Ud, Sd, out=out)
    e1.record(); torch.cuda.synchronize()
    print(B, round(e0.elapsed_time(e1) / 10, 4))
