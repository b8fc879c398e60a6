import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S, synth, Discretizer
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess
from paper_2604_09993_b200.scenario import build_scaling
from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern
for name, kw in (("pointmass_rest", {}), ("biped_walk", {})):
    sc = S.bundled(name, **kw)
    gt = GpuTranscription(sc); dev = gt.device
    z = torch.as_tensor(initial_guess(sc, gt.disc, gt.lay), device=dev)
    asm = SubproblemAssembler(SubproblemPattern(sc, gt.lay, build_scaling(sc, gt.lay)[0]), dev)
    r = gt.linearize_device(z, 1.0)
    x, U, Sv = synth.random_intervals(sc, sc.N - 1, seed=0)
    xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
    out = gt.disc.linearize_batch_device(xd, Ud, Sd)
    def t(fn, n=30):
        for _ in range(5): fn()
        torch.cuda.synchronize(); ts=[]
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        return round(float(np.median(ts))*1e3, 1)
    print(name, "K1 only us", t(lambda: gt.disc.linearize_batch_device(xd, Ud, Sd, out=out)),
          "linearize_all us", t(lambda: gt.linearize_device(z, 1.0, out=r)),
          "assembly us", t(lambda: asm.assemble_device(r, z, reuse=True)))
