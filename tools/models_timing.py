"""One SCP iteration (linearize_all + assembly, device-resident) for every bundled
scenario of the reference's assets: device time per iteration and per interval.  (GPU box)"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.scenario import build_scaling  # noqa: E402
from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern  # noqa: E402

rows = []
for name, kw in (("pointmass_rest", {}), ("monoped_hop", {"N": 20}), ("biped_walk", {}),
                 ("halfcheetah_bound", {"N": 30}), ("halfcheetah_bound", {"N": 200, "substeps": 8})):
    sc = S.bundled(name, **kw)
    gt = GpuTranscription(sc)
    dev = gt.device
    z = torch.as_tensor(initial_guess(sc, gt.disc, gt.lay), device=dev)
    asm = SubproblemAssembler(SubproblemPattern(sc, gt.lay, build_scaling(sc, gt.lay)[0]), dev)
    r = gt.linearize_device(z, 1.0)
    for _ in range(5):
        asm.assemble_device(gt.linearize_device(z, 1.0, out=r), z, reuse=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        asm.assemble_device(gt.linearize_device(z, 1.0, out=r), z, reuse=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    import time

    from paper_2604_09993_b200.subproblem import GpuSCPStep

    step = GpuSCPStep(gt)
    zh = z.cpu().numpy()
    for _ in range(5):
        step.iterate(zh, 1.0)
    t0 = time.perf_counter()
    for _ in range(50):
        step.iterate(zh, 1.0)
    e2e = (time.perf_counter() - t0) / 50 * 1e3
    rows.append({"scenario": name, "N": sc.N, "substeps": sc.substeps, "intervals": sc.N - 1,
                 "ms_per_iteration": ms, "us_per_interval": 1e3 * ms / (sc.N - 1),
                 "e2e_ms_GpuSCPStep": e2e})
    print(rows[-1], flush=True)
json.dump({"note": "device time of linearize_all (K1 || K3) + whole-subproblem assembly (eager launches, device "
                   "events; small models are host-issue bound here), initial guess, median of 30; e2e = wall time of "
                   "GpuSCPStep.iterate (one CUDA graph, host numpy in / scipy program out)",
           "rows": rows}, open("gpurun_out/models_timing.json", "w"), indent=1)
