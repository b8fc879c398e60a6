"""Small fixed workload for ncu captures: HalfCheetah N=30 propagate + linearize (29 intervals)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S, synth, Discretizer
B = int(sys.argv[1]) if len(sys.argv) > 1 else 29
mode = sys.argv[2] if len(sys.argv) > 2 else "both"  # lin | prop | both
sc = S.bundled("halfcheetah_bound", N=30)
g, n_g = sc.path_constraints()
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
x, U, Sv = synth.random_intervals(sc, B, seed=0)
dev = torch.device("cuda")
xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
for _ in range(3):
    if mode in ("prop", "both"):
        disc.propagate_batch_device(xd, Ud, Sd)
    if mode in ("lin", "both"):
        disc.linearize_batch_device(xd, Ud, Sd)
torch.cuda.synchronize()
print("ok")
