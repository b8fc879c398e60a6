"""configs[1]: the reference's own CI-SCVX loop (cito.scp.solve: backtracking
homotopy + host IPM, unchanged) on HalfCheetah N=30 with the GPU drop-ins
installed; per-iteration wall time of each stage.  (GPU box; needs the
reference installed in baseline/_ref -- it runs through the jax shim, test
infrastructure.)  Writes one JSON object to stdout.

  python tools/scp_solve_profile.py [max_iters] [N] [--one-pass]

--one-pass: install_scp (scp_dropin.py) -- the three calls served by one device
pass per iteration -- instead of the three separate drop-ins.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
os.environ.setdefault("CITO_REF_SRC", os.path.join(ROOT, "baseline", "_ref"))

import ref_runner  # noqa: E402

ref_runner.import_cito()
from dataclasses import replace  # noqa: E402

import torch  # noqa: E402
from cito import ocp, scp  # noqa: E402

import paper_2604_09993_b200.linearize as G  # noqa: E402
import paper_2604_09993_b200.subproblem as SP  # noqa: E402
from paper_2604_09993_b200 import install  # noqa: E402

one_pass = "--one-pass" in sys.argv
argv = [a for a in sys.argv[1:] if not a.startswith("--")]
iters = int(argv[0]) if len(argv) > 0 else 3
N = int(argv[1]) if len(argv) > 1 else 30
sc = ocp.load_scenario(os.path.join(ref_runner.assets_dir(), "halfcheetah_bound.json"))
sc = replace(sc, N=N, s_bounds=None)
tr = ocp.get_transcription(sc)
install(tr)
times = {"linearize_all": [], "build_subproblem": [], "precondition": [], "ipm_solve": []}


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        times[name].append(time.perf_counter() - t0)
        return r
    return w


dev_ms = []
if one_pass:
    from paper_2604_09993_b200.scp_dropin import install_scp
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    _orig_replay = torch.cuda.CUDAGraph.replay

    def _timed_replay(g):  # device time of each iteration's graph (CUDA events on the replay stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _orig_replay(g)
        e1.record()
        dev_ms.append((e0, e1))

    torch.cuda.CUDAGraph.replay = _timed_replay
    d = install_scp(scp)
    fns = (scp.linearize_all, scp.build_subproblem, scp.precondition)
else:
    fns = (G.linearize_all, SP.build_subproblem, SP.precondition)
# warm the GPU path (build + first-call setup, graph capture) outside the measured loop
z0 = tr.initial_guess()
for _ in range(2):
    lin = fns[0](tr, z0, 1.0)
    fns[2](fns[1](tr, lin, z0, 1.0, scp.SCPConfig())[0])
del lin  # a result kept alive here would hold one of the step's result slots for the whole run
scp.linearize_all = timed("linearize_all", fns[0])
scp.build_subproblem = timed("build_subproblem", fns[1])
scp.precondition = timed("precondition", fns[2])
scp.ipm_solve = timed("ipm_solve", scp.ipm_solve)
t0 = time.perf_counter()
z, hist, status = scp.solve(sc, scp.SCPConfig(max_iters=iters))
wall = time.perf_counter() - t0
out = {"scenario": f"halfcheetah_bound N={N} (substeps {sc.substeps})", "iterations": len(hist) - 1,
       "status": status, "wall_s": wall,
       "per_iteration_ms": {k: [1e3 * x for x in v] for k, v in times.items()},
       "mean_ms": {k: (1e3 * sum(v) / len(v) if v else None) for k, v in times.items()},
       "delta": [h.delta for h in hist], "j_px": [h.j_px for h in hist], "j_ep": [h.j_ep for h in hist],
       "slots": ({id(t): (len(st._plan["hosts"]), st._plan.get("captures")) for t, st in d._steps.values()}
                 if one_pass else None),
       "graph_device_ms": [a.elapsed_time(b) for a, b in dev_ms[-(len(hist) - 1):]] if dev_ms else None,
       "pre_ipm_ms": [1e3 * (a + b + c) for a, b, c in zip(times["linearize_all"], times["build_subproblem"],
                                                           times["precondition"])],
       "pattern": ({"refetches": sum(st.pattern_refetches for _, st in d._steps.values()),
                    "d2h_bytes": sum(st.d2h_copied for _, st in d._steps.values()),
                    "what": "calls whose CSC pattern moved after a values-only copy (one extra index copy each); "
                            "all device->host bytes of the run incl. warm-up"} if one_pass else None),
       "mode": "install_scp (one device pass per iteration)" if one_pass else "three separate drop-ins",
       "note": "GPU: linearize_all + build_subproblem + precondition (drop-ins); host: the reference's IPM "
               "(cito/_ipm.py) and homotopy, unchanged"}
if one_pass and "--idle-probe" in sys.argv:
    # the same pre-IPM call back to back, after 2.5 s of idling, and after 2.5 s of host
    # numpy work (what the IPM does between two calls): separates GPU idle wake-up from
    # cold host caches in the per-iteration numbers above
    cfg = scp.SCPConfig()

    split = []

    def one():
        t = time.perf_counter()
        lin = scp.linearize_all(tr, z, 0.5)
        t1 = time.perf_counter()
        prog, _ = scp.build_subproblem(tr, lin, z, 0.5, cfg)
        t2 = time.perf_counter()
        scp.precondition(prog)
        t3 = time.perf_counter()
        split.append((t1 - t, t2 - t1, t3 - t2))
        return 1e3 * (t3 - t)

    probe = {"back_to_back": [], "after_idle_2p5s": [], "after_host_work_2p5s": []}
    for _ in range(5):
        split.clear()
        probe["back_to_back"].append(min(one() for _ in range(20)))
        probe.setdefault("back_to_back_split_ms", []).append(
            [round(1e3 * float(np.median([x[i] for x in split])), 4) for i in range(3)])
        time.sleep(2.5)
        probe["after_idle_2p5s"].append(one())
        t_end = time.perf_counter() + 2.5
        M = np.random.default_rng(0).standard_normal((600, 600))
        while time.perf_counter() < t_end:
            M = np.linalg.solve(M + 600 * np.eye(600), M)
        probe["after_host_work_2p5s"].append(one())
    out["idle_probe_ms"] = probe
print(json.dumps(out))
