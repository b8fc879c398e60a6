import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess
from paper_2604_09993_b200.scenario import build_scaling
from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern
dev = torch.device("cuda")
scf = bench.scp_problem(0, fine=True)
gtf = GpuTranscription(scf)
zf = torch.as_tensor(initial_guess(scf, gtf.disc, gtf.lay), device=dev)
asmf = SubproblemAssembler(SubproblemPattern(scf, gtf.lay, build_scaling(scf, gtf.lay)[0]), dev)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
for it in range(12):
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(); r = gtf.linearize_device(zf, 1.0); ev[1].record(); asmf.assemble_device(r, zf); ev[2].record()
    torch.cuda.synchronize()
    print(it, round(ev[0].elapsed_time(ev[1]), 3), round(ev[1].elapsed_time(ev[2]), 3))
