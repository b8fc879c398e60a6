"""K3 (node relations + Jacobians) timing on the configs[3] analogue: 128 HalfCheetah
N=50 initial guesses (6400 nodes, 6272 intervals), L2 flushed; tools/ab.py format."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess_batch  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 128
sc = S.bundled("halfcheetah_bound", N=50)
gt = GpuTranscription(sc)
Z = torch.as_tensor(initial_guess_batch(sc, gt.disc, list(range(P)), gt.lay), device=gt.device)
out = gt.linearize_device(Z, 1.0)
lay = gt.lay
yp = torch.stack([torch.cat([Z[p, lay.y_of_xp(k)], Z[p, lay.y_of_xm(k + 1)]]) for p in range(P)
                  for k in range(lay.N - 1)]).contiguous()
n_q = lay.n_q
tv = torch.stack([torch.cat([Z[p, lay.xm(k)[:n_q]], Z[p, lay.xm(k)[n_q:2 * n_q]], Z[p, lay.xp(k)[n_q:2 * n_q]],
                             Z[p, lay.phi(k)], Z[p, lay.gam(k)]]) for p in range(P) for k in range(lay.N)]).contiguous()
nout = gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=gt.device)
for name, fn, B in (("node", lambda: gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon, out=nout), P * lay.N),
                    ("linearize_all", lambda: gt.linearize_device(Z, 1.0, out=out), P * (lay.N - 1))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"B={B} {name}: {float(np.median(ts)):.4f} ms", flush=True)
