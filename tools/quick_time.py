"""Quick device-resident timing of K1/K2 on synthetic HalfCheetah intervals."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S, synth, Discretizer

import os
sc = S.bundled(os.environ.get("QT_SCENARIO", "halfcheetah_bound"), N=int(os.environ.get("QT_N", "30")))
g, n_g = sc.path_constraints()
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
for B in [int(a) for a in (sys.argv[1:] or ["29", "4096"])]:
    x, U, Sv = synth.random_intervals(sc, B, seed=0)
    dev = torch.device("cuda")
    xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
    out = disc.linearize_batch_device(xd, Ud, Sd)
    torch.cuda.synchronize()
    for name, fn in (("linearize", lambda: disc.linearize_batch_device(xd, Ud, Sd, out=out)),
                     ("propagate", lambda: disc.propagate_batch_device(xd, Ud, Sd))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(f"B={B} {name}: {ms:.3f} ms  -> {B/ms*1e3:.3e} intervals/s", flush=True)
