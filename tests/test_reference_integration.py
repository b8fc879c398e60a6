"""Drop-in test inside the reference's own SCP loop.

The unmodified reference package (installed copy in baseline/_ref, or
/root/reference in the build container) runs through the jax shim
(oracle/jaxshim, test infrastructure); its `cito.scp.linearize_all`,
`build_subproblem`, `precondition` and the transcription's discretizer are
replaced by the GPU implementations and
`cito.scp.solve` runs a few SCP iterations (host IPM + homotopy unchanged).
The iterates must match the reference's own path.  Runs in a subprocess so
the shim's global torch settings cannot leak into other tests.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_src():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "cito")):
            return p
    return None


SCRIPT = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.join(ROOT, "oracle"))
os.environ["CITO_REF_SRC"] = REF
sys.path.insert(0, ROOT)
import ref_runner
cito = ref_runner.import_cito()
from dataclasses import replace
from cito import ocp, scp
import paper_2604_09993_b200.linearize as G
import paper_2604_09993_b200.subproblem as SPB
from paper_2604_09993_b200 import install

name, iters, compare, N, ref_lin, mode = (sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1", int(sys.argv[4]),
                                          sys.argv[5], sys.argv[6])
sc = ocp.load_scenario(os.path.join(REF, "cito", "assets", name + ".json"))
if N:
    sc = replace(sc, N=N, s_bounds=None)
cfg = scp.SCPConfig(max_iters=iters)
out = {}


def oracle_linearize_all(tr, z, delta, jobs=1):
    """cito.scp.linearize_all (scp.py:87-135) with the interval + node linearization of
    the pinned C oracle (test infrastructure): the reference's own path for models
    whose shim linearization (jacfwd under torch.func, ~5 s per interval) is too slow."""
    import pyoracle
    from paper_2604_09993_b200.model import pack_model
    lay = tr.layout
    desc = pack_model(tr.model, tr.mixing, tr.path_fn)
    n = lay.N - 1
    xs = np.stack([z[lay.xp(k)] for k in range(n)])
    us = np.stack([z[lay.u(k)] for k in range(n)])
    ss = np.array([z[lay.s(k)][0] for k in range(n)])
    e, jx, ju, js, bad = pyoracle.linearize(desc, tr.scenario.substeps, xs, us, ss)
    if bad.any():
        raise FloatingPointError("non-finite state during interval integration")
    yp, tv, _ = tr._node_inputs(z)
    psi, pj, th, tj, imp, ij = pyoracle.node_linearize(desc, yp, tv, delta, tr.scenario.ctcs_epsilon)
    defects = np.stack([z[lay.xm(k + 1)] for k in range(n)]) - e
    return scp.LinearizedProblem(z_ref=z, ends=e, jx=jx, ju=ju, js=js, defects=defects, psi=psi, psi_jac=pj,
                                 theta=th, theta_jac=tj, imp_v=imp, imp_jac=ij)


class OracleDisc:
    """propagate() of the pinned oracle for the reference arm's initial_guess."""
    def __init__(self, tr):
        import pyoracle
        from paper_2604_09993_b200.model import pack_model
        self.po, self.desc, self.m = pyoracle, pack_model(tr.model, tr.mixing, tr.path_fn), tr.scenario.substeps

    def propagate(self, xt0, U, S):
        e, bad = self.po.propagate(self.desc, self.m, np.asarray(xt0)[None], np.asarray(U).reshape(1, -1),
                                   np.array([float(S)]))
        if bad.any():
            raise FloatingPointError("non-finite state during interval integration")
        return e[0]


if compare:
    ocp._transcriptions.clear()
    orig = scp.linearize_all
    if ref_lin == "oracle":
        trr = ocp.get_transcription(sc)
        trr.discretizer = OracleDisc(trr)
        scp.linearize_all = oracle_linearize_all
    try:
        z_ref, hist_ref, st_ref = scp.solve(sc, cfg)
    finally:
        scp.linearize_all = orig
    out["ref"] = [h.z.tolist() for h in hist_ref]
    out["ref_delta"] = [h.delta for h in hist_ref]
    out["ref_jpx"] = [h.j_px for h in hist_ref]
    out["ref_jep"] = [h.j_ep for h in hist_ref]
ocp._transcriptions.clear()
tr = ocp.get_transcription(sc)
install(tr)                       # tr.discretizer -> GPU (initial_guess uses it)
import time
orig = scp.linearize_all, scp.build_subproblem, scp.precondition
if mode == "scp":  # one device pass per iteration (paper_2604_09993_b200.scp_dropin)
    from paper_2604_09993_b200.scp_dropin import install_scp
    drop = install_scp(scp)
    fns = (scp.linearize_all, scp.build_subproblem, scp.precondition)
else:
    fns = (G.linearize_all,           # GPU linearize_all (intervals + node relations)
           SPB.build_subproblem,       # GPU subproblem assembly (CSC values, b, h)
           SPB.precondition)           # GPU row scaling of the assembled program
pre_ipm = []


def timed(f):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        pre_ipm.append(time.perf_counter() - t0)
        return r
    return w


scp.linearize_all, scp.build_subproblem, scp.precondition = (timed(f) for f in fns)
try:
    z, hist, st = scp.solve(sc, cfg)
finally:
    scp.linearize_all, scp.build_subproblem, scp.precondition = orig
out["pre_ipm_ms"] = [1e3 * (pre_ipm[3 * i] + pre_ipm[3 * i + 1] + pre_ipm[3 * i + 2]) for i in range(len(pre_ipm) // 3)]
out["gpu"] = [h.z.tolist() for h in hist]
out["gpu_delta"] = [h.delta for h in hist]
out["gpu_jpx"] = [h.j_px for h in hist]
out["gpu_jep"] = [h.j_ep for h in hist]
out["status"] = st
out["launches"] = tr.discretizer.launch_count() + (G._cache[id(tr)][1].disc.launch_count() if mode != "scp"
                                                   else drop._step(tr).gt.disc.launch_count())
print("RESULT " + json.dumps(out))
'''


def _run(name, iters, compare, N=0, ref_lin="shim", mode="three", timeout=1500):
    ref = _ref_src()
    if ref is None:
        pytest.skip("reference package not available (baseline/_ref or /root/reference)")
    code = f"ROOT = {ROOT!r}\nREF = {ref!r}\n" + SCRIPT
    p = subprocess.run([sys.executable, "-c", code, name, str(iters), "1" if compare else "0", str(N), ref_lin, mode], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert p.returncode == 0 and line, p.stderr[-3000:]
    return json.loads(line[0][7:])


@pytest.mark.gpu
def test_scp_solve_pointmass_matches_reference_path():
    import numpy as np

    r = _run("pointmass_rest", 4, True)
    assert len(r["gpu"]) == len(r["ref"])
    for zg, zr in zip(r["gpu"], r["ref"]):
        zg, zr = np.asarray(zg), np.asarray(zr)
        assert np.max(np.abs(zg - zr)) <= 1e-6 * (1.0 + np.max(np.abs(zr)))
    assert np.allclose(r["gpu_delta"], r["ref_delta"], rtol=1e-9)
    assert r["launches"] > 0


@pytest.mark.gpu
def test_scp_solve_halfcheetah_n30_matches_reference_path():
    """configs[1]: HalfCheetah N=30, the reference's cito.scp.solve (backtracking
    homotopy + host IPM, scp.py:383-467) for 3 iterations, once on its own path
    (reference build_subproblem/precondition, linearization by the pinned oracle
    port, which matches the reference's jacfwd to <= 1e-11) and once with the
    three GPU drop-ins installed: every iterate, delta and progress measure agree."""
    import numpy as np

    r = _run("halfcheetah_bound", 3, True, N=30, ref_lin="oracle")
    _check_halfcheetah(r)


@pytest.mark.gpu
def test_scp_solve_halfcheetah_n30_one_pass_dropins():
    """Same, with install_scp: linearize_all + build_subproblem + precondition of every
    iteration served by one CUDA-graph replay and one D2H (scp_dropin.py).  Records
    the pre-IPM wall time per iteration."""
    r = _run("halfcheetah_bound", 3, True, N=30, ref_lin="oracle", mode="scp")
    _check_halfcheetah(r)
    assert len(r["pre_ipm_ms"]) == 3 and r["launches"] > 0
    print("pre-IPM ms per iteration (install_scp):", r["pre_ipm_ms"])


def _check_halfcheetah(r):
    import numpy as np

    assert len(r["gpu"]) == len(r["ref"]) == 4
    for zg, zr in zip(r["gpu"], r["ref"]):
        zg, zr = np.asarray(zg), np.asarray(zr)
        assert np.all(np.isfinite(zg))
        assert np.max(np.abs(zg - zr)) <= 1e-6 * (1.0 + np.max(np.abs(zr)))
    assert np.allclose(r["gpu_delta"], r["ref_delta"], rtol=1e-9)
    assert np.allclose(r["gpu_jpx"], r["ref_jpx"], rtol=1e-5, atol=1e-9)
    assert np.allclose(r["gpu_jep"], r["ref_jep"], rtol=1e-5, atol=1e-9)
