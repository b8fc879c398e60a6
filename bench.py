#!/usr/bin/env python
"""Benchmark of the B200 discretize+linearize hot path (one JSON line on rank 0).

Metric (BASELINE.json): interval linearizations/sec (fp64), HalfCheetah N=30;
SCP-iteration linearize ms (= ms_per_step).

Workload ``scp`` (default, configs[1]): one SCP iteration's linearization of
HalfCheetah (halfcheetah_bound.json, N=30, 5 substeps -> 29 intervals) at an
SCP-realistic point (the scenario's initial guess; rank r uses seed r):
gather from z -> K1 interval linearize (ends, Phi, B-, B+, dS) -> defects ->
K3 node relations + Jacobians -> K4 scatter of the dynamics rows into CSC
values + b.  ``batch``: configs[2], 4096 independent synthetic intervals per
GPU (one K1 launch per step).

  value  device-resident throughput (inputs already in HBM), CUDA events per
         step on the launching stream, L2 flushed (256 MiB write) between steps,
         max over ranks.
  e2e    same step through the public API with host buffers: H2D of z (pinned)
         + device work + D2H of every output (LinearizedProblem arrays, CSC
         values, b) inside the timed region.
  --impl reference   the reference algorithm on the host cores: the C oracle
         port (oracle/cito_oracle.c; JAX, the reference's runtime, is not
         installable here), all threads, same workload/metric.

Multi-GPU: one process per GPU (torchrun); each rank linearizes its own
independent problem(s) (weak scaling), no data-path collective.
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "interval linearizations/sec (fp64) HalfCheetah N=30; SCP-iteration linearize ms"
UNIT = "intervals/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["scp", "fine", "batch", "multistart"], default="scp")
    p.add_argument("--no-fine-extra", action="store_true")
    p.add_argument("--problems", type=int, default=128, help="multistart: problems per GPU (configs[3]: 1024 / 8)")
    p.add_argument("--batch", type=int, default=4096)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--sample-seconds", type=float, default=None, help="reference arm: time-bounded sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-batch-extra", action="store_true")
    return p.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# --------------------------------------------------------------------------- shared problem setup
FINE = dict(N=200, substeps=8)  # configs[4]: HalfCheetah fine grid (the reference has no RK4: its RKF at 8 substeps)


def scp_problem(seed, fine=False):
    from paper_2604_09993_b200 import scenario as S

    sc = S.bundled("halfcheetah_bound", **(FINE if fine else dict(N=30)))
    sc.seed = seed
    return sc


class _OracleDisc:
    """propagate() through the CPU oracle: builds the reference-arm input (the
    scenario's initial guess) without touching the GPU path."""

    def __init__(self, sc):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle

        from paper_2604_09993_b200.model import pack_model

        g, n_g = sc.path_constraints()
        self.po, self.desc, self.substeps = pyoracle, pack_model(sc.model, sc.mixing_matrix(n_g), g), sc.substeps

    def propagate(self, xt0, U, S):
        e = self.po.propagate(self.desc, self.substeps, np.asarray(xt0)[None], np.asarray(U).reshape(1, -1),
                              np.array([float(S)]))[0]
        return e[0]


def _reference_scp():
    """The reference's own Python (cito.scp/ocp/conic, installed in baseline/_ref) via the
    jax shim, for the host-side subproblem assembly; None when not installed."""
    src = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(src, "cito")):
        return None
    os.environ["CITO_REF_SRC"] = src
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import ref_runner

        ref_runner.import_cito()
        from cito import ocp, scp

        return ocp, scp
    except Exception:
        return None


def cpu_step_fn(sc, seed):
    """One SCP iteration's pre-IPM work on the host: the reference's linearization
    algorithm via the oracle port (intervals + node relations) and, when the
    reference is installed, its own build_subproblem + canonicalize."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    from paper_2604_09993_b200.linearize import node_inputs
    from paper_2604_09993_b200.model import pack_model
    from paper_2604_09993_b200.scenario import Layout

    lay = Layout(sc)
    g, n_g = sc.path_constraints()
    desc = pack_model(sc.model, sc.mixing_matrix(n_g), g)
    from paper_2604_09993_b200.linearize import initial_guess

    z = initial_guess(sc, _OracleDisc(sc), lay)
    starts = np.stack([z[lay.xp(k)] for k in range(lay.N - 1)])
    Us = np.stack([z[lay.u(k)] for k in range(lay.N - 1)])
    Ss = np.array([z[lay.s(k)][0] for k in range(lay.N - 1)])
    yp, tv = node_inputs(lay, z)
    ref = _reference_scp()
    tr = None
    if ref is not None:
        from dataclasses import replace

        ocp, scp = ref
        rsc = ocp.load_scenario(os.path.join(ROOT, "tests", "golden", "assets", "halfcheetah_bound.json"))
        tr = ocp.Transcription(replace(rsc, N=sc.N, s_bounds=None, substeps=sc.substeps))
    step_fn.with_assembly = tr is not None

    def step():
        e, jx, ju, js, _ = pyoracle.linearize(desc, sc.substeps, starts, Us, Ss)
        psi, pj, th, tj, imp, ij = pyoracle.node_linearize(desc, yp, tv, 1.0, sc.ctcs_epsilon)
        if tr is not None:
            defects = np.stack([z[lay.xm(k + 1)] for k in range(lay.N - 1)]) - e
            lin = scp.LinearizedProblem(z_ref=z, ends=e, jx=jx, ju=ju, js=js, defects=defects, psi=psi, psi_jac=pj,
                                        theta=th, theta_jac=tj, imp_v=imp, imp_jac=ij)
            scp.build_subproblem(tr, lin, z, 1.0, scp.SCPConfig())
        return lay.N - 1

    return step, pyoracle


def step_fn():
    pass


def cpu_batch_fn(sc, B):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    from paper_2604_09993_b200 import synth
    from paper_2604_09993_b200.model import pack_model

    g, n_g = sc.path_constraints()
    desc = pack_model(sc.model, sc.mixing_matrix(n_g), g)
    x, U, S = synth.random_intervals(sc, B, seed=0)

    def step():
        pyoracle.linearize(desc, sc.substeps, x, U, S)
        return B

    return step, pyoracle


def time_cpu(step, seconds, min_steps=1):
    n, t0 = 0, time.perf_counter()
    units = 0
    while n < min_steps or time.perf_counter() - t0 < seconds:
        units += step()
        n += 1
    dt = time.perf_counter() - t0
    return units / dt, n, dt


# --------------------------------------------------------------------------- GPU helpers
class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.count(",") >= 8]
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows]
        mx = float(rows[0][2])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if "Active" in v and "Not" not in v})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].strip() not in ("", "[N/A]"))}


def fp64_peak_tflops(torch, dev):
    from paper_2604_09993_b200 import _lib

    out = torch.zeros(1, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    best = 0.0
    for iters in (64, 2048, 2048, 2048, 2048):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fl = _lib.lib().cito_dfma_peak(iters, out.data_ptr(), s.cuda_stream)
        e1.record(s)
        s.synchronize()
        best = max(best, fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def flops_per_interval(key):
    path = os.path.join(ROOT, "profiles", "flops_per_interval.json")
    if not os.path.exists(path):
        return None, None
    d = json.load(open(path))
    e = d.get(key)
    return (e["flops"], d.get("definition")) if e else (None, None)


def ncu_traffic(key):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    return json.load(open(path)).get(key, {}).get("dram_bytes_per_launch")


def run_ours(args):
    import torch

    rank, world, local = env_rank()
    dist = None
    # CITO_BENCH_BACKEND=gloo + CITO_BENCH_DEVICE=0 exercise the multi-rank code path
    # with several ranks on one GPU (test only: no kernel waits on another rank)
    backend = os.environ.get("CITO_BENCH_BACKEND", "nccl")
    if os.environ.get("CITO_BENCH_DEVICE") is not None:
        local = int(os.environ["CITO_BENCH_DEVICE"])
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group(backend)
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    from paper_2604_09993_b200 import synth
    from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess
    from paper_2604_09993_b200.scenario import build_scaling
    from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern, build_subproblem

    fine = args.workload == "fine"
    sc = scp_problem(seed=rank, fine=fine)
    gt = GpuTranscription(sc, device=dev.index)
    lay = gt.lay
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    # --- SCP-iteration workload state
    z = initial_guess(sc, gt.disc, lay)
    z_dev = torch.as_tensor(z, device=dev)
    delta = 1.0
    scale_v, state_scale, u_scale = build_scaling(sc, lay)
    asm = SubproblemAssembler(SubproblemPattern(sc, lay, scale_v), dev)
    n_int = lay.N - 1

    k1_ev = []

    lin_out = gt.linearize_device(z_dev, delta)  # output buffers reused by every step

    def scp_step(zd, record=False):
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r = gt.linearize_device(zd, delta, k1_events=(e0, e1), out=lin_out)
            k1_ev.append((e0, e1))
        else:
            r = gt.linearize_device(zd, delta, out=lin_out)
        asm.assemble_device(r, zd, reuse=True)  # whole subproblem: CSC of A, G (+ zero compaction), b, h
        return r

    # --- batch workload state
    if args.workload == "batch" or (args.workload == "scp" and not args.no_batch_extra):
        B = args.batch
        ok = lambda x, u, s: synth.well_posed(gt.disc.propagate_batch_device(
            *(torch.as_tensor(a, device=dev) for a in (x, u, s)))[0].cpu().numpy())
        xb, Ub, Sb, redrawn = synth.random_intervals(sc, B, seed=100 + rank, finite_fn=ok)
        xb_d, Ub_d, Sb_d = (torch.as_tensor(a, device=dev) for a in (xb, Ub, Sb))
        bout = gt.disc.linearize_batch_device(xb_d, Ub_d, Sb_d)

    def batch_step(record=False):
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        gt.disc.linearize_batch_device(xb_d, Ub_d, Sb_d, out=bout)
        if record:
            e1.record(stream)
            k1_ev.append((e0, e1))

    if args.workload == "multistart":
        # configs[3] analogue: HalfCheetah N=50 multi-start initial guesses (no quadruped
        # exists in the reference); each rank owns `problems` starts
        from paper_2604_09993_b200 import scenario as S2
        from paper_2604_09993_b200.parallel import gather_rows

        sc50 = S2.bundled("halfcheetah_bound", N=50)
        gt50 = GpuTranscription(sc50, device=dev.index)
        from paper_2604_09993_b200.linearize import initial_guess_batch

        seeds = [rank * args.problems + i for i in range(args.problems)]
        Z = initial_guess_batch(sc50, gt50.disc, seeds, gt50.lay)  # batched multi-start generation (§8(f) 4)
        Z_dev = torch.as_tensor(Z, device=dev)
        ms_out = gt50.linearize_device(Z_dev, 1.0)

        def ms_step(record=False):
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                gt50.linearize_device(Z_dev, 1.0, k1_events=(e0, e1), out=ms_out)
                k1_ev.append((e0, e1))
            else:
                gt50.linearize_device(Z_dev, 1.0, out=ms_out)
            # result collection: per-problem max |defect| to every rank (NCCL all_gather at N > 1)
            metric = ms_out["defects"].view(args.problems, -1).abs().amax(dim=1)
            return gather_rows(metric) if dist else metric

    def timed(step_fn, K, W):
        for _ in range(W):
            step_fn(False)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        k1_ev.clear()
        evs = []
        launches0 = _lib_launches()
        for _ in range(K):
            flush.zero_()  # L2 flush outside the timed events
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step_fn(True)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        launches = _lib_launches() - launches0
        ms = float(np.sum([a.elapsed_time(b) for a, b in evs]))
        k1_ms = float(np.mean([a.elapsed_time(b) for a, b in k1_ev]))
        if dist:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, k1_ms, launches

    K, W = args.steps, max(3, args.warmup)
    clocks = Clocks(dev.index if world == 1 else local)
    step_k1_ms = None
    if args.workload in ("scp", "fine"):
        ms_tot, k1_ms, launches = timed(lambda rec: scp_step(z_dev, rec), K, W)
        # the interval kernel alone (the roofline kernel; in the step it overlaps K3 and
        # includes the fork/join): same intervals, device-resident, events on its stream
        zh = z_dev.cpu().numpy()
        xs = torch.as_tensor(np.stack([zh[lay.xp(k)] for k in range(n_int)]), device=dev)
        us = torch.as_tensor(np.stack([zh[lay.u(k)] for k in range(n_int)]), device=dev)
        ss = torch.as_tensor(np.array([zh[lay.s(k)][0] for k in range(n_int)]), device=dev)
        kout = gt.disc.linearize_batch_device(xs, us, ss)
        for _ in range(W):
            gt.disc.linearize_batch_device(xs, us, ss, out=kout)
        kev = []
        for _ in range(K):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gt.disc.linearize_batch_device(xs, us, ss, out=kout)
            e1.record(stream)
            kev.append((e0, e1))
        torch.cuda.synchronize()
        step_k1_ms = k1_ms
        k1_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
        units_per_step, B_k1 = n_int, n_int
    elif args.workload == "multistart":
        gt.disc = gt50.disc  # launch counter of the handle actually used
        ms_tot, k1_ms, launches = timed(ms_step, K, W)
        units_per_step = B_k1 = args.problems * (sc50.N - 1)
    else:
        ms_tot, k1_ms, launches = timed(batch_step, K, W)
        units_per_step, B_k1 = args.batch, args.batch
    clk = clocks.stop()
    ms_per_step = ms_tot / K
    value = world * units_per_step * K / (ms_tot * 1e-3)

    extra = {}
    if args.workload == "scp" and not args.no_batch_extra:
        bms, bk1, _ = timed(batch_step, max(5, K // 5), 3)
        nb = max(5, K // 5)
        extra["batch_extra"] = {"workload": f"HalfCheetah synthetic batch of {args.batch} intervals (configs[2])",
                                "value": args.batch * nb / (bms * 1e-3), "unit": UNIT, "ms_per_step": bms / nb,
                                "k1_ms": bk1}

    if args.workload == "scp" and not args.no_fine_extra:
        # configs[4]: HalfCheetah N=200, 8 substeps, one SCP iteration (K1 + K3 + assembly)
        scf = scp_problem(seed=rank, fine=True)
        gtf = GpuTranscription(scf, device=dev.index)
        zf = torch.as_tensor(initial_guess(scf, gtf.disc, gtf.lay), device=dev)
        asmf = SubproblemAssembler(SubproblemPattern(scf, gtf.lay, build_scaling(scf, gtf.lay)[0]), dev)

        fine_out = gtf.linearize_device(zf, delta)

        def fine_step(record=False):
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                r = gtf.linearize_device(zf, delta, k1_events=(e0, e1), out=fine_out)
                k1_ev.append((e0, e1))
            else:
                r = gtf.linearize_device(zf, delta, out=fine_out)
            asmf.assemble_device(r, zf, reuse=True)

        nf = max(5, K // 5)
        fms, fk1, _ = timed(fine_step, nf, 5)
        extra["fine_extra"] = {"workload": "HalfCheetah N=200, 8 RKF substeps, one SCP iteration (configs[4]; "
                                           "the reference has no RK4)",
                               "value": (scf.N - 1) * nf / (fms * 1e-3), "unit": UNIT, "ms_per_step": fms / nf,
                               "k1_ms": fk1}

    # --- e2e through the public API with host (pinned) buffers
    if args.workload in ("scp", "fine"):
        # public API of one SCP iteration's pre-IPM work (= cito.scp.linearize_all +
        # build_subproblem, scp.py:412-413): host numpy z in, host scipy ConicProgram out
        from paper_2604_09993_b200.subproblem import GpuSCPStep

        scp_api = GpuSCPStep(gt)

        def e2e_step():
            return scp_api.iterate(z, delta)

        e2e_step()
        h2d = z.nbytes + 16  # z plus [delta, epsilon] (one pinned H2D per step)
        d2h = scp_api.d2h_bytes()  # packed D2H per step: fixed fields + the CSC arrays up to their caps
    elif args.workload == "multistart":
        Z_pin = torch.as_tensor(Z).pin_memory()
        ms_host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True).numpy() for k, v in ms_out.items()}

        def e2e_step():
            # public multi-start API: host Z in, host arrays out (caller-owned page-locked
            # buffers); chunks of ~one K1 wave, each copied back while the next computes
            return gt50.linearize_to_host(Z_pin, 1.0, out=ms_host)

        e2e_step()
        h2d = Z.nbytes
        d2h = int(sum(v.numel() * v.element_size() for v in ms_out.values()))
    else:
        xb_p, Ub_p, Sb_p = (torch.as_tensor(a).pin_memory() for a in (xb, Ub, Sb))
        bouts = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in bout]

        xb_n, Ub_n, Sb_n = (t.numpy() for t in (xb_p, Ub_p, Sb_p))
        outs_n = tuple(t.numpy() for t in bouts[:4])

        def e2e_step():
            # public drop-in Discretizer.linearize_batch (augmentation.py:236-242): host
            # arrays in, host arrays out (caller-owned page-locked buffers); the C entry
            # copies the inputs up and pipelines the results back chunk by chunk
            return gt.disc.linearize_batch(xb_n, Ub_n, Sb_n, out=outs_n)

        e2e_step()
        h2d = xb.nbytes + Ub.nbytes + Sb.nbytes
        d2h = int(sum(t.numel() * t.element_size() for t in bout[:4])) + 4 * args.batch  # + per-interval flags
    for _ in range(W):
        e2e_step()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(K):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * units_per_step * K / e2e_s

    peak = fp64_peak_tflops(torch, dev)
    key = "halfcheetah_s8" if fine else "halfcheetah_s5"
    F, fdef = flops_per_interval(key)
    achieved = F * B_k1 / (k1_ms * 1e-3) / 1e12 if F else None
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": ncu_traffic(f"k_linearize_{'scp' if fine else args.workload}"),
                "kernel": ("k_linearize2<Topo_halfcheetah_g2,1> (1 interval/CTA)" if B_k1 <= 98
                           else "k_linearize<Topo_halfcheetah_g2,1,2> (2 intervals/CTA in lockstep)" if B_k1 <= 246
                           else "k_linearize<Topo_halfcheetah_g2,1,3> (3 intervals/CTA in lockstep)"),
                "kernel_ms": k1_ms, "intervals_per_launch": B_k1,
                "step_linearize_all_ms": step_k1_ms,
                "flops_per_interval": F, "flops_definition": fdef,
                "peak_source": "measured in this run: FP64 DFMA probe kernel (cito_dfma_peak); MEASURED_PEAKS.json "
                               "has no fp64 entry"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference arm itself, in a subprocess (isolates the jax shim), time-bounded sample
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference", "--workload", args.workload,
                            "--sample-seconds", str(args.cpu_seconds), "--warmup", "1", "--problems",
                            str(args.problems), "--batch", str(args.batch)], capture_output=True, text=True,
                           cwd=ROOT, env={k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE")})
        lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
        cpu = json.loads(lines[-1])["cpu_baseline"] if lines else {"error": p.stderr[-400:]}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic" if args.workload == "batch" else "synthetic (scenario initial guess, seed=rank)",
        "config": {"workload": {"scp": "scp: one SCP-iteration linearize of HalfCheetah N=30 (halfcheetah_bound.json, "
                                       "5 RKF substeps, 29 intervals; K1+K3 + whole-subproblem assembly)",
                                "fine": "fine: one SCP-iteration linearize of HalfCheetah N=200, 8 RKF substeps "
                                        "(configs[4]; 199 intervals; K1+K3 + whole-subproblem assembly)",
                                "batch": f"batch: {args.batch} independent synthetic HalfCheetah intervals per GPU "
                                         "(configs[2])",
                                "multistart": f"multistart: {args.problems} HalfCheetah N=50 initial guesses per GPU "
                                              "(configs[3] analogue), linearize_all (K1+K3) + NCCL all_gather of "
                                              "per-problem defect norms"}[args.workload],
                   "intervals_per_step_per_gpu": units_per_step, "l2": "flushed (256 MiB write) between timed steps",
                   "parallelism": f"replicas x{world} (independent problems per rank, no collective)"},
        "roofline": roofline, "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_s / K * 1e3},
        "gpu_launches": int(launches), "clocks": clk,
    }
    line.update(extra)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_reference(args):
    rank, world, local = env_rank()
    if rank != 0:
        return
    sc = scp_problem(seed=0, fine=args.workload == "fine")
    if args.workload in ("scp", "fine", "multistart"):
        step, po = cpu_step_fn(sc, 0)
        sample = (f"HalfCheetah N={sc.N} ({sc.substeps} substeps) initial-guess SCP iteration per step: oracle-port "
                  f"linearization ({sc.N - 1} intervals + node relations)" + (" + the reference's own build_subproblem/canonicalize (baseline/_ref)"
                                         if step_fn.with_assembly else " (reference not installed: no assembly)"))
    else:
        B = max(8, min(args.batch, 256))
        step, po = cpu_batch_fn(sc, B)
        sample = f"{B} synthetic HalfCheetah intervals per step (bounded sample of the {args.batch}-interval batch)"
    for _ in range(max(1, args.warmup)):
        step()
    t0 = time.perf_counter()
    units, n = 0, 0
    while (n < args.steps) if args.sample_seconds is None else (n < 1 or time.perf_counter() - t0 < args.sample_seconds):
        units += step()
        n += 1
    dt = time.perf_counter() - t0
    v = units / dt
    sample += f"; {n} steps in {dt:.1f} s on {os.cpu_count()} host cores"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": n, "warmup": args.warmup,
            "ms_per_step": dt / n * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": args.workload, "note": "reference algorithm on host cores via the C oracle port; "
                       "the reference's JAX runtime is not installable (no jax wheel, no network)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": po.get_threads(), "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _lib_launches():
    """Kernels launched by libcito_b200 so far (C ABI counter + CUDA-graph replays)."""
    from paper_2604_09993_b200 import _lib

    return _lib.launch_count()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

