"""K1 time vs batch size around wave boundaries (HalfCheetah, 5 substeps), for the
batch-kernel dispatch.  (GPU box)  python tools/tail_probe.py B1 B2 ...
Env switches of cito_capi.cu (CITO_K1, CITO_K1_IPC2_MAX, ...) apply per process."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import Discretizer, scenario as S, synth  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
g, n_g = sc.path_constraints()
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
dev = torch.device("cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
out_rows = {}
for B in [int(a) for a in sys.argv[1:]]:
    x, U, Sv = synth.random_intervals(sc, B, seed=0)
    xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
    out = disc.linearize_batch_device(xd, Ud, Sd)
    for _ in range(3):
        disc.linearize_batch_device(xd, Ud, Sd, out=out)
    ms = []
    for _ in range(15):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        disc.linearize_batch_device(xd, Ud, Sd, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    out_rows[B] = round(sorted(ms)[len(ms) // 2], 4)
print(json.dumps(out_rows))
