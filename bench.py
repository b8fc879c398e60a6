#!/usr/bin/env python
"""Benchmark of the B200 discretize+linearize hot path (one JSON line on rank 0).

Metric (BASELINE.json): interval linearizations/sec (fp64), HalfCheetah N=30;
SCP-iteration linearize ms (= ms_per_step).

Workloads (``--workload``):
  scp (default, configs[1])  one SCP iteration's pre-IPM work for HalfCheetah
        (halfcheetah_bound.json, N=30, 5 RKF substeps -> 29 intervals) at the
        scenario's initial guess (rank r: seed r): K1 interval linearization +
        defects and K3 node relations (one linearize_all call, cito/scp.py:87-135),
        then the whole-subproblem CSC assembly with exact-zero compaction + b/h
        (cito/scp.py:160-351 + cito/conic.py:209-269).  At N > 1 GPUs: replicas
        (one independent problem per rank, no collective).
  batch (configs[2])   B (default 4096) independent synthetic HalfCheetah
        intervals, split in contiguous ranges over the ranks (strong scaling),
        the full results gathered to rank 0's GPU with one grouped NCCL
        send/recv inside the timed step (paper_2604_09993_b200.parallel).
  multistart (configs[3] analogue)  P (default 1024) HalfCheetah N=50 initial
        guesses (no quadruped exists in the reference), whole problems per rank,
        linearize_all of each rank's problems in one call + NCCL gather of all
        LinearizedProblem arrays to rank 0.
  fine (configs[4])    as scp with N=200, 8 RKF substeps.

Line fields:
  value  whole-job throughput, inputs resident in HBM: CUDA events on the
         launching stream per step, L2 flushed (256 MiB write) between steps,
         max over ranks.
  e2e    the same metric through the public API with host buffers:
         scp/fine: GpuSCPStep.iterate -- upload of [z, delta, epsilon, ...] from pinned memory, the
           device step whose last kernels write the assembled program into a
           pinned host buffer (CSC values and column pointers, b, h, flags; the
           CSC row indices only when that buffer does not hold the current
           sparsity pattern -- the compaction flags a moved pattern); the
           returned LinearizedProblem stays device-backed (lazy:
           cito.scp.solve only hands it to build_subproblem), so its Jacobians
           are not copied (h2d/d2h bytes per step are reported).
         batch: Discretizer.linearize_batch (N=1) / ShardedBatch.linearize(...,
           collect="host") (N>1): host arrays in, every Jacobian back on the host.
         multistart: GpuTranscription.linearize_to_host / ShardedMultiStart(...,
           collect="host"): host arrays of every LinearizedProblem field.
  roofline  the dominant kernel (K1) timed alone with CUDA events: counted
         algorithmic fp64 flops / time / the DFMA peak measured in this run
         (frac), and the ncu-executed fp64 instruction flops (frac_executed).
  cpu_baseline  the reference arm's line (``--impl reference``) run in a
         subprocess on rank 0: the reference algorithm on the host cores
         (oracle port for the linearization, the reference's own Python for the
         subproblem assembly) -- "iteration" leg and "linearize_only" leg.

``--impl reference``: the reference's CPU implementation of the same workload
(the C oracle port, oracle/cito_oracle.c, all host threads; JAX, the reference's
runtime, is not installable here), same config/metric/unit; N>1: rank 0 only.
``--gpus N`` without torchrun re-launches itself under torch.distributed.run.
"""

import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "interval linearizations/sec (fp64) HalfCheetah N=30; SCP-iteration linearize ms"
UNIT = "intervals/s"
FINE = dict(N=200, substeps=8)  # configs[4]: the reference has no RK4; its RKF at 8 substeps


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["scp", "fine", "batch", "multistart"], default="scp")
    p.add_argument("--no-fine-extra", action="store_true")
    p.add_argument("--no-batch-extra", action="store_true")
    p.add_argument("--problems", type=int, default=1024, help="multistart: problems in total (configs[3]: 1024)")
    p.add_argument("--batch", type=int, default=4096, help="batch: intervals in total (configs[2]: 4096)")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--sample-seconds", type=float, default=None, help="reference arm: time-bounded sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def relaunch_under_torchrun(args):
    """``bench.py --gpus N`` started without torchrun: run N ranks (one per GPU) the
    way the driver does, with the same arguments."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, cwd=ROOT))


def config_for(args, world):
    """The `config` dict of both arms (identical for the same arguments)."""
    wl = args.workload
    desc = {
        "scp": "scp: one SCP-iteration linearize of HalfCheetah N=30 (halfcheetah_bound.json, 5 RKF substeps, "
               "29 intervals; K1+K3 + whole-subproblem assembly) at the scenario's initial guess",
        "fine": "fine: one SCP-iteration linearize of HalfCheetah N=200, 8 RKF substeps (configs[4]; 199 intervals; "
                "K1+K3 + whole-subproblem assembly) at the scenario's initial guess",
        "batch": f"batch: {args.batch} independent synthetic HalfCheetah intervals in total (configs[2]), "
                 "split over the GPUs, results gathered to rank 0",
        "multistart": f"multistart: {args.problems} HalfCheetah N=50 initial guesses in total (configs[3] "
                      "analogue), linearize_all (K1+K3) split over the GPUs, results gathered to rank 0",
    }[wl]
    per = {"scp": 29, "fine": 199, "batch": args.batch, "multistart": args.problems * 49}[wl]
    par = (f"replicas x{world} (an independent problem per rank, no collective)" if wl in ("scp", "fine")
           else f"shards x{world} (contiguous ranges per rank; one grouped NCCL send/recv to rank 0 for result "
                "collection)" if world > 1 else "single GPU")
    return {"workload": desc, "intervals_per_step": per * (world if wl in ("scp", "fine") else 1),
            "l2": "flushed (256 MiB write) between timed steps", "parallelism": par}


# --------------------------------------------------------------------------- shared problem setup
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


class CpuIteration:
    """One SCP iteration's pre-IPM work on the host: the reference's linearization
    algorithm via the oracle port (intervals + node relations) and, when the
    reference is installed, its own build_subproblem + canonicalize."""

    def __init__(self, sc):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle

        from paper_2604_09993_b200.linearize import initial_guess, node_inputs
        from paper_2604_09993_b200.model import pack_model
        from paper_2604_09993_b200.scenario import Layout

        self.po, self.sc = pyoracle, sc
        lay = self.lay = Layout(sc)
        g, n_g = sc.path_constraints()
        self.desc = pack_model(sc.model, sc.mixing_matrix(n_g), g)
        z = self.z = initial_guess(sc, _OracleDisc(sc), lay)
        n = lay.N - 1
        self.starts = np.stack([z[lay.xp(k)] for k in range(n)])
        self.Us = np.stack([z[lay.u(k)] for k in range(n)])
        self.Ss = np.array([z[lay.s(k)][0] for k in range(n)])
        self.yp, self.tv = node_inputs(lay, z)
        ref = _reference_scp()
        self.tr = None
        if ref is not None:
            from dataclasses import replace

            ocp, self.scp = ref
            rsc = ocp.load_scenario(os.path.join(ROOT, "tests", "golden", "assets", "halfcheetah_bound.json"))
            self.tr = ocp.Transcription(replace(rsc, N=sc.N, s_bounds=None, substeps=sc.substeps))

    def linearize(self):
        e, jx, ju, js, _ = self.po.linearize(self.desc, self.sc.substeps, self.starts, self.Us, self.Ss)
        node = self.po.node_linearize(self.desc, self.yp, self.tv, 1.0, self.sc.ctcs_epsilon)
        return e, jx, ju, js, node

    def iteration(self):
        e, jx, ju, js, (psi, pj, th, tj, imp, ij) = self.linearize()
        if self.tr is not None:
            lay, z, scp = self.lay, self.z, self.scp
            defects = np.stack([z[lay.xm(k + 1)] for k in range(lay.N - 1)]) - e
            lin = scp.LinearizedProblem(z_ref=z, ends=e, jx=jx, ju=ju, js=js, defects=defects, psi=psi, psi_jac=pj,
                                        theta=th, theta_jac=tj, imp_v=imp, imp_jac=ij)
            scp.build_subproblem(self.tr, lin, z, 1.0, scp.SCPConfig())
        return self.lay.N - 1


def time_cpu(step, seconds=None, steps=None):
    n, units, t0 = 0, 0, time.perf_counter()
    while (n < steps) if seconds is None else (n < 1 or time.perf_counter() - t0 < seconds):
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
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if "Active" in v and "Not" not in v})
        pw = [float(r[3]) for r in rows if r[3].strip() not in ("", "[N/A]")]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(pw) if pw else None}


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


def _profile_json(name):
    path = os.path.join(ROOT, "profiles", name)
    return json.load(open(path)) if os.path.exists(path) else {}


def flops_per_interval(key):
    d = _profile_json("flops_per_interval.json")
    e = d.get(key)
    return (e["flops"], d.get("definition")) if e else (None, None)


def executed_flops_per_interval(B):
    """ncu-executed fp64 flops per interval (DFMA = 2) of the K1 generation that serves
    a batch of B intervals (profiles/fp64_instruction_counts.json)."""
    d = _profile_json("fp64_instruction_counts.json")
    key = "latency" if B <= 98 else "batch"
    e = d.get(key)
    return (e["executed_fp64_flops_per_interval"], e.get("source")) if e else (None, None)


def ncu_traffic(key):
    return _profile_json("ncu_summary.json").get(key, {}).get("dram_bytes_per_launch")


def _lib_launches():
    """Kernels launched by libcito_b200 so far (C ABI counter + CUDA-graph replays)."""
    from paper_2604_09993_b200 import _lib

    return _lib.launch_count()


def k1_kernel_name(B):
    return ("k_linearize2<Topo_halfcheetah_g2,1> (1 interval/CTA)" if B <= 98
            else "k_linearize<Topo_halfcheetah_g2,1,2> (2 intervals/CTA in lockstep)" if B <= 246
            else "k_linearize<Topo_halfcheetah_g2,1,3> (3 intervals/CTA in lockstep)")


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
    from paper_2604_09993_b200.parallel import HostResult, ShardedBatch, ShardedMultiStart, gather_slices, shard_range
    from paper_2604_09993_b200.scenario import build_scaling
    from paper_2604_09993_b200.subproblem import GpuSCPStep, SubproblemAssembler, SubproblemPattern

    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    k1_ev = []
    K, W = args.steps, max(3, args.warmup)

    def ev_pair():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(step_fn, K, W):
        """W warm-up steps, then K steps bracketed by barrier + synchronize; per-step
        CUDA events on the launching stream (L2 flush outside them); max over ranks."""
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
            flush.zero_()
            e0, e1 = ev_pair()
            e0.record(stream)
            step_fn(True)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        launches = _lib_launches() - launches0
        ms = float(np.sum([a.elapsed_time(b) for a, b in evs]))
        k1_ms = float(np.mean([a.elapsed_time(b) for a, b in k1_ev])) if k1_ev else None
        if dist:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, k1_ms, launches

    def kernel_alone(disc, xs, us, ss, reps):
        """K1 alone (the roofline kernel), device-resident, events on its stream."""
        kout = disc.linearize_batch_device(xs, us, ss)
        for _ in range(3):
            disc.linearize_batch_device(xs, us, ss, out=kout)
        kev = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = ev_pair()
            e0.record(stream)
            disc.linearize_batch_device(xs, us, ss, out=kout)
            e1.record(stream)
            kev.append((e0, e1))
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b) for a, b in kev]))

    def scp_setup(fine, seed):
        sc = scp_problem(seed=seed, fine=fine)
        gt = GpuTranscription(sc, device=dev.index)
        z = initial_guess(sc, gt.disc, gt.lay)
        z_dev = torch.as_tensor(z, device=dev)
        asm = SubproblemAssembler(SubproblemPattern(sc, gt.lay, build_scaling(sc, gt.lay)[0]), dev)
        out = gt.linearize_device(z_dev, 1.0)  # output buffers reused by every step

        def step(record=False):
            if record:
                e0, e1 = ev_pair()
                r = gt.linearize_device(z_dev, 1.0, k1_events=(e0, e1), out=out)
                k1_ev.append((e0, e1))
            else:
                r = gt.linearize_device(z_dev, 1.0, out=out)
            asm.assemble_device(r, z_dev, reuse=True)  # whole subproblem: CSC of A, G (+ zero compaction), b, h
        return sc, gt, z, z_dev, step

    def batch_setup(B):
        """configs[2]: B intervals in total, rank r linearizes its contiguous range into
        rank 0's full arrays (NCCL gather)."""
        sc = scp_problem(seed=0)
        gt = GpuTranscription(sc, device=dev.index)
        ok = lambda x, u, s: synth.well_posed(gt.disc.propagate_batch_device(  # noqa: E731
            *(torch.as_tensor(a, device=dev) for a in (x, u, s)))[0].cpu().numpy())
        xb, Ub, Sb, _ = synth.random_intervals(sc, B, seed=100, finite_fn=ok)
        lo, hi = shard_range(B, rank, world)
        sb = ShardedBatch(gt.disc, device=dev)
        x_d, U_d, S_d = (torch.as_tensor(a, device=dev) for a in (xb, Ub, Sb))
        sb.compute(x_d, U_d, S_d)  # allocate

        def step(record=False):
            out, _, _ = sb.compute(x_d, U_d, S_d)
            if dist is not None and world > 1:
                if record:
                    c0, c1 = ev_pair()
                    c0.record(stream)
                sb._collect(out, B, lo, "device", None)
                if record:
                    c1.record(stream)
                    k1_ev.append((c0, c1))
        return gt, sb, xb, Ub, Sb, (lo, hi), step

    clocks = Clocks(dev.index)
    extra = {}
    wl = args.workload
    if wl in ("scp", "fine"):
        fine = wl == "fine"
        sc, gt, z, z_dev, step = scp_setup(fine, rank)
        lay = gt.lay
        n_int = lay.N - 1
        ms_tot, step_k1_ms, launches = timed(step, K, W)
        units_per_step = n_int * world
        zh = z
        xs = torch.as_tensor(np.stack([zh[lay.xp(k)] for k in range(n_int)]), device=dev)
        us = torch.as_tensor(np.stack([zh[lay.u(k)] for k in range(n_int)]), device=dev)
        ss = torch.as_tensor(np.array([zh[lay.s(k)][0] for k in range(n_int)]), device=dev)
        k1_ms = kernel_alone(gt.disc, xs, us, ss, K)
        B_k1 = n_int
        extra["linearize_only"] = {"value": n_int * world / (step_k1_ms * 1e-3), "unit": UNIT,
                                   "ms_per_step": step_k1_ms,
                                   "what": "linearize_all alone (K1 + K3 + defects, one C call) inside the step"}
        scp_api = GpuSCPStep(gt)

        def e2e_step():
            return scp_api.iterate(z, 1.0)

        e2e_step()
        h2d = z.nbytes + 40  # z plus [delta, epsilon, stamp, two flags], uploaded from pinned memory per step
        d2h = None  # counted over the timed steps (GpuSCPStep.d2h_copied): fixed fields + CSC values, + the
        # CSC row indices in a step whose result buffer does not hold the current pattern
        e2e_note = "GpuSCPStep.iterate: host z in, host scipy program out; LinearizedProblem device-backed (lazy)"
    elif wl == "batch":
        B = args.batch
        gt, sb, xb, Ub, Sb, (lo, hi), step = batch_setup(B)
        ms_tot, collect_ms, launches = timed(step, K, W)
        units_per_step = B
        xs, us, ss = (torch.as_tensor(a[lo:hi], device=dev) for a in (xb, Ub, Sb))
        k1_ms = kernel_alone(gt.disc, xs, us, ss, K)
        B_k1 = hi - lo
        if collect_ms is not None:
            extra["collect"] = {"nccl_gather_ms": collect_ms, "what": "grouped NCCL send/recv of every rank's "
                                "ends/jx/ju/js/flags into rank 0's full device arrays (device time on rank 0's stream)"}
        host = HostResult(sb.shapes(B)) if world > 1 else None
        bout = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).numpy() for t in sb._alloc(B).values()][:4]

        def e2e_step():
            if world > 1:
                return sb.linearize(xb, Ub, Sb, collect="host", host=host)
            return gt.disc.linearize_batch(xb, Ub, Sb, out=tuple(bout))

        e2e_step()
        h2d = (xb.nbytes + Ub.nbytes + Sb.nbytes) // world
        n, nu2 = gt.disc.n_xt, 2 * gt.disc.n_u
        d2h = (B * 8 * (2 * n + n * n + n * nu2) + 4 * B) // world
        e2e_note = ("Discretizer.linearize_batch: host arrays in, all four result arrays back on the host"
                    if world == 1 else "ShardedBatch.linearize(collect='host'): every rank H2D its rows, "
                    "linearizes, D2H into one shared page-locked host result (the N-parallel-D2H collection)")
    else:  # multistart
        from paper_2604_09993_b200 import scenario as S2

        sc50 = S2.bundled("halfcheetah_bound", N=50)
        ms = ShardedMultiStart(sc50, list(range(args.problems)), device=dev)
        gt = ms.gt
        B_loc = (ms.hi - ms.lo) * (sc50.N - 1)

        def step(record=False):
            if record:
                e0, e1 = ev_pair()
                e0.record(stream)
            ms.compute(1.0)
            if record:
                e1.record(stream)
            if dist is not None and world > 1:
                gather_slices(ms.out, ms.full, ms.rows, ms.all_bounds)
            if record:
                k1_ev.append((e0, e1))

        ms_tot, lin_ms, launches = timed(step, K, W)
        units_per_step = args.problems * (sc50.N - 1)
        lay = gt.lay
        xs = torch.as_tensor(np.concatenate([np.stack([z[lay.xp(k)] for k in range(lay.N - 1)]) for z in ms.Z]),
                             device=dev)
        us = torch.as_tensor(np.concatenate([np.stack([z[lay.u(k)] for k in range(lay.N - 1)]) for z in ms.Z]),
                             device=dev)
        ss = torch.as_tensor(np.concatenate([np.array([z[lay.s(k)][0] for k in range(lay.N - 1)]) for z in ms.Z]),
                             device=dev)
        k1_ms = kernel_alone(gt.disc, xs, us, ss, K)
        B_k1 = B_loc
        host = HostResult(ms.shapes()) if world > 1 else None
        ms_host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True).numpy() for k, v in ms.out.items()}
        Z_pin = torch.as_tensor(ms.Z).pin_memory()

        def e2e_step():
            if world > 1:
                return ms.linearize(1.0, collect="host", host=host)
            return gt.linearize_to_host(Z_pin, 1.0, out=ms_host)

        e2e_step()
        h2d = ms.Z.nbytes
        d2h = int(sum(v.numel() * v.element_size() for v in ms.out.values()))
        e2e_note = ("GpuTranscription.linearize_to_host: host Z in, every LinearizedProblem array back on the host"
                    if world == 1 else "ShardedMultiStart.linearize(collect='host'): per-rank D2H into one shared "
                    "page-locked host result")
    clk = clocks.stop()
    ms_per_step = ms_tot / K
    value = units_per_step * K / (ms_tot * 1e-3)

    # --- extras: configs[2] batch beside the scp headline; configs[4] fine grid
    if wl == "scp" and not args.no_batch_extra:
        B = args.batch
        _, _, _, _, _, (blo, bhi), bstep = batch_setup(B)
        nb = max(5, K // 5)
        bms, bcoll, _ = timed(bstep, nb, 3)
        extra["batch_extra"] = {"workload": f"HalfCheetah synthetic batch of {B} intervals (configs[2])"
                                + (f", split over {world} GPUs + NCCL gather to rank 0" if world > 1 else ""),
                                "value": B * nb / (bms * 1e-3), "unit": UNIT, "ms_per_step": bms / nb,
                                "nccl_gather_ms": bcoll}
    if wl == "scp" and not args.no_fine_extra:
        _, gtf, _, _, fstep = scp_setup(True, rank)
        nf = max(5, K // 5)
        fms, fk1, _ = timed(fstep, nf, 5)
        extra["fine_extra"] = {"workload": "HalfCheetah N=200, 8 RKF substeps, one SCP iteration (configs[4]; "
                                           "the reference has no RK4)",
                               "value": (gtf.lay.N - 1) * world * nf / (fms * 1e-3), "unit": UNIT,
                               "ms_per_step": fms / nf, "linearize_all_ms": fk1}

    # --- e2e through the public API with host buffers
    for _ in range(W):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    c0 = scp_api.d2h_copied if wl in ("scp", "fine") else 0
    t0 = time.perf_counter()
    for _ in range(K):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    if d2h is None:
        d2h = (scp_api.d2h_copied - c0) / K
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = units_per_step * K / e2e_s

    peak = fp64_peak_tflops(torch, dev)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    F, fdef = flops_per_interval("halfcheetah_s8" if wl == "fine" else "halfcheetah_s5")
    Fx, fxsrc = executed_flops_per_interval(B_k1) if wl != "fine" else (None, None)
    achieved = F * B_k1 / (k1_ms * 1e-3) / 1e12 if F else None
    achieved_x = Fx * B_k1 / (k1_ms * 1e-3) / 1e12 if Fx else None
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": ncu_traffic(f"k_linearize_{'scp' if wl == 'fine' else wl}"),
                "kernel": k1_kernel_name(B_k1), "kernel_ms": k1_ms, "intervals_per_launch": B_k1,
                "flops_per_interval": F, "flops_definition": fdef,
                "achieved_executed": achieved_x, "frac_executed": (achieved_x / peak) if achieved_x else None,
                # the latency kernel runs one CTA per interval: with fewer intervals than SMs only
                # B_k1 of the SMs carry work, so the same time against their share of the peak
                "frac_of_busy_sms": ((achieved / (peak * min(1.0, B_k1 / n_sm))) if achieved and B_k1 <= 98 else None),
                "executed_flops_per_interval": Fx, "executed_source": fxsrc,
                "peak_source": "measured in this run: FP64 DFMA probe kernel (cito_dfma_peak); MEASURED_PEAKS.json "
                               "has no fp64 entry"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference arm itself, in a subprocess (isolates the jax shim), time-bounded sample
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference", "--workload", wl,
                            "--sample-seconds", str(args.cpu_seconds), "--warmup", "1", "--problems",
                            str(args.problems), "--batch", str(args.batch)], capture_output=True, text=True,
                           cwd=ROOT, env={k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE")})
        lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
        cpu = json.loads(lines[-1])["cpu_baseline"] if lines else {"error": p.stderr[-400:]}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if wl in ("scp", "fine") else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic" if wl == "batch" else "synthetic (scenario initial guess; scp: seed = rank)",
        "config": config_for(args, world),
        "roofline": roofline, "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_s / K * 1e3, "api": e2e_note},
        "gpu_launches": int(launches), "clocks": clk,
    }
    line.update(extra)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    rank, world, local = env_rank()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    wl = args.workload
    legs = {}
    if wl in ("scp", "fine"):
        it = CpuIteration(scp_problem(seed=0, fine=wl == "fine"))
        n_int = it.lay.N - 1
        it.iteration()
        what = (f"HalfCheetah N={it.sc.N} ({it.sc.substeps} substeps) initial-guess SCP iteration per step: oracle-port "
                f"linearization ({n_int} intervals + node relations)")
        what += (" + the reference's own build_subproblem/canonicalize (baseline/_ref)" if it.tr is not None
                 else " (reference not installed: no assembly)")
        secs = args.sample_seconds
        v, n, dt = time_cpu(it.iteration, secs, None if secs else args.steps)
        lv, ln, ldt = time_cpu(lambda: (it.linearize(), n_int)[1], secs / 2 if secs else None,
                               None if secs else args.steps)
        legs["iteration"] = {"value": v, "ms_per_step": dt / n * 1e3, "steps": n}
        legs["linearize_only"] = {"value": lv, "ms_per_step": ldt / ln * 1e3, "steps": ln,
                                  "what": "oracle-port linearize_batch + node relations only (no assembly)"}
        if it.tr is not None and wl == "scp":
            # the reference's own linearize_batch (unmodified source) through the jax -> torch.func
            # shim, a tiny sample: eager per-element AD, far slower than JAX/XLA would be -- context
            # only, never the headline
            import torch

            torch.set_num_threads(os.cpu_count() or 1)
            xs, us, ss = it.starts[:1], it.Us[:1], it.Ss[:1]
            it.tr.discretizer.linearize_batch(xs, us, ss)
            sv, sn, sdt = time_cpu(lambda: (it.tr.discretizer.linearize_batch(xs, us, ss), 1)[1], None, 1)
            legs["reference_source_shim"] = {"value": sv, "ms_per_step": sdt / sn * 1e3, "steps": sn,
                                             "what": "cito.augmentation.Discretizer.linearize_batch of 1 interval, "
                                                     "unmodified reference source under the jax->torch.func shim "
                                                     f"({torch.get_num_threads()} torch threads)"}
        sample = f"{what}; {n} steps in {dt:.1f} s"
    elif wl == "batch":
        sc = scp_problem(seed=0)
        from paper_2604_09993_b200 import synth
        from paper_2604_09993_b200.model import pack_model

        g, n_g = sc.path_constraints()
        desc = pack_model(sc.model, sc.mixing_matrix(n_g), g)
        Bs = max(8, min(args.batch, 256))
        x, U, S = synth.random_intervals(sc, Bs, seed=100)

        def step():
            pyoracle.linearize(desc, sc.substeps, x, U, S)
            return Bs

        step()
        v, n, dt = time_cpu(step, args.sample_seconds, None if args.sample_seconds else args.steps)
        legs["linearize_only"] = {"value": v, "ms_per_step": dt / n * 1e3, "steps": n}
        sample = f"{Bs} synthetic HalfCheetah intervals per step (bounded sample of the {args.batch}-interval batch); " \
                 f"{n} steps in {dt:.1f} s"
    else:
        from paper_2604_09993_b200 import scenario as S2
        from paper_2604_09993_b200.linearize import initial_guess_batch, node_inputs
        from paper_2604_09993_b200.model import pack_model
        from paper_2604_09993_b200.scenario import Layout

        sc = S2.bundled("halfcheetah_bound", N=50)
        lay = Layout(sc)
        g, n_g = sc.path_constraints()
        desc = pack_model(sc.model, sc.mixing_matrix(n_g), g)
        P = max(1, min(args.problems, 4))
        Z = initial_guess_batch(sc, _OracleBatchDisc(sc), list(range(P)), lay)
        n = lay.N - 1

        def step():
            for z in Z:
                pyoracle.linearize(desc, sc.substeps, np.stack([z[lay.xp(k)] for k in range(n)]),
                                   np.stack([z[lay.u(k)] for k in range(n)]),
                                   np.array([z[lay.s(k)][0] for k in range(n)]))
                yp, tv = node_inputs(lay, z)
                pyoracle.node_linearize(desc, yp, tv, 1.0, sc.ctcs_epsilon)
            return P * n

        step()
        v, n_s, dt = time_cpu(step, args.sample_seconds, None if args.sample_seconds else args.steps)
        legs["linearize_only"] = {"value": v, "ms_per_step": dt / n_s * 1e3, "steps": n_s}
        sample = f"{P} of the {args.problems} HalfCheetah N=50 starts per step (bounded sample): oracle-port " \
                 f"linearize_all; {n_s} steps in {dt:.1f} s"
    head = legs.get("iteration", legs["linearize_only"])
    v = head["value"]
    sample += f" on {pyoracle.get_threads()} of {os.cpu_count()} host cores"
    cpu_model = None
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), None)
    except OSError:
        pass
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": head["steps"],
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "weak" if wl in ("scp", "fine") else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic" if wl == "batch" else "synthetic (scenario initial guess; scp: seed = rank)",
            "impl": "reference", "config": config_for(args, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": pyoracle.get_threads(), "kind": "port",
                             "cpu_model": cpu_model, "sample": sample, "legs": legs,
                             "note": "reference algorithm on host cores via the C oracle port (dense forward-mode "
                                     "duals like jacfwd, LU like jnp.linalg.solve); the reference's JAX runtime is "
                                     "not installable (no jax wheel, no network)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class _OracleBatchDisc(_OracleDisc):
    def propagate_batch(self, xt0s, Us, Ss):
        return self.po.propagate(self.desc, self.substeps, np.asarray(xt0s), np.asarray(Us), np.asarray(Ss))[0]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
