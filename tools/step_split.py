"""Device-time split of the bench's scp step: linearize_all (K1 || K3) vs the assembly.  (GPU box)"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.scenario import build_scaling  # noqa: E402
from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
gt = GpuTranscription(sc)
dev = gt.device
z = torch.as_tensor(initial_guess(sc, gt.disc, gt.lay), device=dev)
asm = SubproblemAssembler(SubproblemPattern(sc, gt.lay, build_scaling(sc, gt.lay)[0]), dev)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
r = gt.linearize_device(z, 1.0)
for _ in range(5):
    asm.assemble_device(gt.linearize_device(z, 1.0, out=r), z)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
t_lin, t_asm, t_all = [], [], []
for _ in range(50):
    flush.zero_()
    e0, e1, e2 = ev(), ev(), ev()
    e0.record()
    gt.linearize_device(z, 1.0, out=r)
    e1.record()
    asm.assemble_device(r, z)
    e2.record()
    torch.cuda.synchronize()
    t_lin.append(e0.elapsed_time(e1))
    t_asm.append(e1.elapsed_time(e2))
    t_all.append(e0.elapsed_time(e2))
# assembly alone with the device idle before it (host issue latency excluded)
t_asm2 = []
for _ in range(50):
    torch.cuda.synchronize()
    torch.cuda._sleep(200000)
    e1, e2 = ev(), ev()
    e1.record()
    asm.assemble_device(r, z)
    e2.record()
    torch.cuda.synchronize()
    t_asm2.append(e1.elapsed_time(e2))
med = lambda x: round(float(np.median(x)) * 1e3, 1)  # noqa: E731
print("us: linearize_all", med(t_lin), "assembly", med(t_asm), "step", med(t_all), "assembly (pre-queued)", med(t_asm2))
