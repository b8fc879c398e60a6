"""Throughput of K1 vs batch size (HalfCheetah, 5 substeps): intervals/s and fraction
of the measured fp64 peak, device-resident inputs, CUDA events.  (GPU box)
Writes one JSON object to stdout."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2604_09993_b200 import Discretizer, scenario as S, synth  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
g, n_g = sc.path_constraints()
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
dev = torch.device("cuda")
F = json.load(open(os.path.join(".", "profiles", "flops_per_interval.json")))["halfcheetah_s5"]["flops"]
peak = bench.fp64_peak_tflops(torch, dev)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
rows = []
for B in (1, 29, 148, 296, 592, 1184, 2368, 4096, 8192, 16384, 50176):
    x, U, Sv = synth.random_intervals(sc, B, seed=0)
    xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
    out = disc.linearize_batch_device(xd, Ud, Sd)
    for _ in range(3):
        disc.linearize_batch_device(xd, Ud, Sd, out=out)
    ms = []
    for _ in range(5 if B > 4096 else 10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        disc.linearize_batch_device(xd, Ud, Sd, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    m = sorted(ms)[len(ms) // 2]
    rows.append({"B": B, "ms": m, "intervals_per_s": B / (m * 1e-3),
                 "fp64_frac": F * B / (m * 1e-3) / 1e12 / peak})
    del out, xd, Ud, Sd
    torch.cuda.empty_cache()
print(json.dumps({"workload": "HalfCheetah linearize_batch (5 RKF substeps), device-resident, L2 flushed",
                  "fp64_peak_tflops_measured": peak, "flops_per_interval": F, "rows": rows}))
