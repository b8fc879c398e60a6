"""Do K1 (29 intervals) and K3 (N=30 node items) overlap when launched on two streams?
Prints the device time of K1 alone, K3 alone and both (K1 on the current stream, K3
on a second stream, joined)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
dev = gt.device
z = torch.as_tensor(initial_guess(sc, gt.disc, gt.lay), device=dev)
lay = gt.lay
zh = z.cpu().numpy()
n = lay.N - 1
xs = torch.as_tensor(np.stack([zh[lay.xp(k)] for k in range(n)]), device=dev)
us = torch.as_tensor(np.stack([zh[lay.u(k)] for k in range(n)]), device=dev)
ss = torch.as_tensor(np.array([zh[lay.s(k)][0] for k in range(n)]), device=dev)
kout = gt.disc.linearize_batch_device(xs, us, ss)
yp, tv = z[gt._i_yp].contiguous(), z[gt._i_th].contiguous()
nout = gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon)
main = torch.cuda.Stream()
side = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)


def timed(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(main):
            e0.record(main)
            fn()
            e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def k1():
    gt.disc.linearize_batch_device(xs, us, ss, out=kout, stream=main.cuda_stream)


def k3():
    gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon, out=nout, stream=main.cuda_stream)


def both(k3_first=False):
    def run():
        side.wait_stream(main)
        if k3_first:
            gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon, out=nout, stream=side.cuda_stream)
            gt.disc.linearize_batch_device(xs, us, ss, out=kout, stream=main.cuda_stream)
        else:
            gt.disc.linearize_batch_device(xs, us, ss, out=kout, stream=main.cuda_stream)
            gt.nodes.device(yp, tv, 1.0, sc.ctcs_epsilon, out=nout, stream=side.cuda_stream)
        main.wait_stream(side)
    return run


for name, fn in (("k1", k1), ("k3", k3), ("both_k1_first", both()), ("both_k3_first", both(True)),
                 ("linearize_all", lambda: gt.linearize_device(z, 1.0))):
    for _ in range(3):
        with torch.cuda.stream(main):
            fn()
    print(f"{name}: {timed(fn):.4f} ms", flush=True)
