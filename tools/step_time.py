"""Device time of one SCP iteration of HalfCheetah N=30 (L2 flushed), printed in the
tools/ab.py format: linearize_all (K1 + K3, one C call) and the whole step
(+ subproblem assembly)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.scenario import build_scaling  # noqa: E402
from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern  # noqa: E402

for N in [int(a) for a in (sys.argv[1:] or ["30"])]:
    sc = S.bundled("halfcheetah_bound", N=N, **({"substeps": 8} if N >= 200 else {}))
    gt = GpuTranscription(sc)
    dev = gt.device
    z = torch.as_tensor(initial_guess(sc, gt.disc, gt.lay), device=dev)
    asm = SubproblemAssembler(SubproblemPattern(sc, gt.lay, build_scaling(sc, gt.lay)[0]), dev)
    out = gt.linearize_device(z, 1.0)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def lin():
        gt.linearize_device(z, 1.0, out=out)

    lay = gt.lay
    zh = z.cpu().numpy()
    xs = torch.as_tensor(np.stack([zh[lay.xp(k)] for k in range(N - 1)]), device=dev)
    us = torch.as_tensor(np.stack([zh[lay.u(k)] for k in range(N - 1)]), device=dev)
    ss = torch.as_tensor(np.array([zh[lay.s(k)][0] for k in range(N - 1)]), device=dev)
    kout = gt.disc.linearize_batch_device(xs, us, ss)
    yp_i = gt._i_yp
    th_i = gt._i_th

    def k1():
        gt.disc.linearize_batch_device(xs, us, ss, out=kout)

    yp = z[yp_i].contiguous()
    tv = z[th_i].contiguous()
    nout = gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon)

    def k3():
        gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon, out=nout)

    def step():
        r = gt.linearize_device(z, 1.0, out=out)
        asm.assemble_device(r, z, reuse=True)

    for name, fn in (("k1_alone", k1), ("k3_alone", k3), ("linearize_all", lin), ("step", step)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"B={N - 1} {name}: {float(np.median(ts)):.4f} ms", flush=True)
