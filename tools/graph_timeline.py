"""Device timeline of GpuSCPStep.iterate's graph replay (torch.profiler / CUPTI):
every kernel and copy of one replay with its start offset and duration.  (GPU box)

  python tools/graph_timeline.py [--precondition] [--fine] [--bare]
"""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2604_09993_b200 import scenario as S  # noqa: E402
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess  # noqa: E402
from paper_2604_09993_b200.subproblem import GpuSCPStep  # noqa: E402

fine = "--fine" in sys.argv
sc = S.bundled("halfcheetah_bound", N=200 if fine else 30)
if fine:
    from dataclasses import replace

    sc = replace(sc, substeps=8)
gt = GpuTranscription(sc)
z = initial_guess(sc, gt.disc, gt.lay)
step = GpuSCPStep(gt)
pc = "--precondition" in sys.argv
for _ in range(20):
    step.iterate(z, 1.0, precondition=pc)
torch.cuda.synchronize()
R = 10
bare = "--bare" in sys.argv  # replay the captured graph alone (no host work around it)
g_bare = step._plan["hosts"][0].graphs[pc]
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(R):
        if bare:
            g_bare.replay()
            torch.cuda.synchronize()
        else:
            step.iterate(z, 1.0, precondition=pc)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
# split into replays at gaps > 20 us
groups, cur = [], []
for e in ev:
    if cur and e.time_range.start - max(c.time_range.end for c in cur) > 20:
        groups.append(cur)
        cur = []
    cur.append(e)
groups.append(cur)
g = groups[len(groups) // 2]
t0 = g[0].time_range.start
print(f"{len(groups)} replays; median replay span (us):",
      np.median([max(e.time_range.end for e in gg) - gg[0].time_range.start for gg in groups]))
for e in g:
    print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:90]}")
