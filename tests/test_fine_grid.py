"""configs[4]: HalfCheetah N=200 with 8 RKF substeps (the reference has no RK4).

Golden `halfcheetah_n200s8.npz` (tests/golden/make_golden_fine.py): the
reference's own initial guess, the reference's build_subproblem -> canonicalize
(cito/scp.py:160-351, cito/conic.py:209-269) and precondition
(cito/conic.py:281-338) of the oracle's linearization there, and 4 synthetic
intervals linearized by the reference itself at 8 substeps.

The assembly at N=200 has 3,904 CSC column blocks per matrix -- more than the
B200 holds resident at once -- so these tests exercise the one-pass
compaction's look-back across non-resident blocks, repeatedly (graph replays).
"""

import numpy as np
import pytest
import scipy.sparse as sp

import pyoracle
from conftest import golden_scenario, load_golden, rel_err, scenario_desc

NAME = "halfcheetah_n200s8"
TOL = 1e-9


def _lin(g):
    return {"jx": g["ig_jx"], "ju": g["ig_ju"], "js": g["ig_js"], "ends": g["ig_ends"], "imp_jac": g["ig_imp_jac"],
            "theta_jac": g["ig_theta_jac"], "psi_jac": g["ig_psi_jac"], "imp_v": g["ig_imp"], "theta": g["ig_theta"],
            "psi": g["ig_psi"], "z_ref": g["ig_z"]}


def _ig_batch(lay, z):
    n = lay.N - 1
    return (np.stack([z[lay.xp(k)] for k in range(n)]), np.stack([z[lay.u(k)] for k in range(n)]),
            np.array([z[lay.s(k)][0] for k in range(n)]))


def test_oracle_matches_reference_at_8_substeps():
    """The oracle (which generated ig_*) against the reference's own linearize_batch at 8 substeps."""
    g = load_golden(NAME)
    sc = golden_scenario(NAME)
    assert sc.N == 200 and sc.substeps == 8
    e, jx, ju, js, bad = pyoracle.linearize(scenario_desc(sc), sc.substeps, g["lin_xt0"], g["lin_U"], g["lin_S"])
    assert not bad.any()
    for a, k in ((e, "ends"), (jx, "jx"), (ju, "ju"), (js, "js")):
        assert rel_err(a, g[f"lin_{k}"]) <= 1e-11, k
        assert np.array_equal(a == 0.0, g[f"lin_{k}"] == 0.0), k


def test_recipes_reproduce_reference_csc_n200():
    """CPU restatement of the device recipes reproduces the reference CSC bit-exactly."""
    from paper_2604_09993_b200.scenario import Layout, build_scaling
    from paper_2604_09993_b200.subproblem import SubproblemPattern
    from test_subproblem import _eval_numpy, _rhs_numpy

    g = load_golden(NAME)
    sc = golden_scenario(NAME)
    lay = Layout(sc)
    pat = SubproblemPattern(sc, lay, build_scaling(sc, lay)[0])
    lin = _lin(g)
    for M, rows in (("A", pat.lin_rows_A), ("G", pat.lin_rows_G)):
        csc = getattr(pat, M)
        indptr, indices, data = _eval_numpy(pat, csc, lin)
        assert tuple(g[f"sp0_{M}_shape"]) == (csc["nrows"], pat.n)
        assert np.array_equal(indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(indices, g[f"sp0_{M}_indices"])
        assert np.array_equal(data, g[f"sp0_{M}_data"]), M
        rhs = _rhs_numpy(pat, csc, rows, lin)
        assert rel_err(rhs, g["sp0_b"] if M == "A" else g["sp0_h"]) <= 1e-13, M
    assert pat.n_orthant == int(g["sp0_nonneg"]) and pat.soc_dims == tuple(g["sp0_soc"])
    assert np.array_equal(pat.objective_c(g["sp0_zj"]), g["sp0_c"])
    nb = -(-pat.n // 32)
    assert nb > 1184  # more column blocks than 148 SMs x 8 resident CTAs


@pytest.mark.gpu
def test_gpu_linearize_all_n200_vs_golden():
    """K1 (199 intervals, 8 substeps; golden: oracle) + K3 (golden: the reference's own
    node Jacobians, whose rounding residues the exact-zero pattern must reproduce) at
    the reference's initial guess, per interval / node."""
    import torch

    from paper_2604_09993_b200.linearize import GpuTranscription

    g = load_golden(NAME)
    sc = golden_scenario(NAME)
    gt = GpuTranscription(sc)
    r = gt.linearize_device(torch.as_tensor(g["ig_z"], device=gt.device), 1.0)
    torch.cuda.synchronize()
    for k, gk in (("ends", "ig_ends"), ("jx", "ig_jx"), ("ju", "ig_ju"), ("js", "ig_js"), ("defects", "ig_defects"),
                  ("psi_jac", "ig_psi_jac"), ("theta_jac", "ig_theta_jac"), ("imp_jac", "ig_imp_jac"),
                  ("psi", "ig_psi"), ("theta", "ig_theta"), ("imp_v", "ig_imp")):
        a, b = r[k].cpu().numpy(), g[gk]
        worst = max(rel_err(a[i], b[i]) for i in range(a.shape[0]))
        assert worst <= TOL, (k, worst)
        if k.endswith("jac") or k in ("jx", "ju", "js"):
            assert np.array_equal(a == 0.0, b == 0.0), k


@pytest.mark.gpu
def test_gpu_linearize_batch_vs_reference_8_substeps():
    from paper_2604_09993_b200 import Discretizer

    g = load_golden(NAME)
    sc = golden_scenario(NAME)
    gg, n_g = sc.path_constraints()
    d = Discretizer(sc.model, mixing=sc.mixing_matrix(n_g), path_fn=gg, substeps=sc.substeps)
    out = d.linearize_batch(g["lin_xt0"], g["lin_U"], g["lin_S"])
    for a, k in zip(out, ("ends", "jx", "ju", "js")):
        assert rel_err(a, g[f"lin_{k}"]) <= TOL, k


@pytest.mark.gpu
@pytest.mark.parametrize("precondition", [False, True])
def test_gpu_assembly_n200_bit_exact(precondition):
    """Device assembly from the golden linearization: the reference's CSC bit for bit,
    five times in a row on the same assembler (the look-back workspace is reused)."""
    import torch

    from paper_2604_09993_b200.scenario import Layout, build_scaling
    from paper_2604_09993_b200.subproblem import LIN_SOURCES, SubproblemAssembler, SubproblemPattern

    g = load_golden(NAME)
    sc = golden_scenario(NAME)
    lay = Layout(sc)
    dev = torch.device("cuda")
    asm = SubproblemAssembler(SubproblemPattern(sc, lay, build_scaling(sc, lay)[0]), dev)
    lin = _lin(g)
    lin_dev = {k: torch.as_tensor(np.ascontiguousarray(lin[k], dtype=np.float64), device=dev) for k in LIN_SOURCES}
    z_dev = torch.as_tensor(lin["z_ref"], device=dev)
    for _ in range(5):
        out = asm.assemble_device(lin_dev, z_dev, precondition=precondition, reuse=True)
        res = asm.to_program(out, g["sp0_zj"])
        prog = res[0]
        for M in ("A", "G"):
            mat = getattr(prog, M)
            assert np.array_equal(mat.indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(mat.indices,
                                                                                      g[f"sp0_{M}_indices"]), M
            ref = g[f"pcsp0_{M}_data"] if precondition else g[f"sp0_{M}_data"]
            assert np.array_equal(mat.data, ref), M
        if precondition:
            prec = res[1]
            assert np.array_equal(prec.row_scale_A, g["pcsp0_row_scale_A"])
            assert np.array_equal(prec.row_scale_G, g["pcsp0_row_scale_G"])
            assert rel_err(prog.b, g["pcsp0_b"]) <= 1e-13 and rel_err(prog.h, g["pcsp0_h"]) <= 1e-13
        else:
            assert rel_err(prog.b, g["sp0_b"]) <= 1e-13 and rel_err(prog.h, g["sp0_h"]) <= 1e-13


@pytest.mark.gpu
def test_gpu_scp_step_n200_matches_reference():
    """The public one-iteration API at configs[4]: pattern bit-exact, values rel <= 1e-9,
    over several graph replays (plain and preconditioned)."""
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    g = load_golden(NAME)
    step = GpuSCPStep(golden_scenario(NAME))
    for it in range(4):
        pc = it % 2 == 1
        res = step.iterate(g["ig_z"], 1.0, precondition=pc)
        lin, prog = res[0], res[1]
        for M in ("A", "G"):
            mat = getattr(prog, M)
            assert np.array_equal(mat.indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(mat.indices,
                                                                                      g[f"sp0_{M}_indices"]), M
            mat = sp.csc_matrix(mat)
            ref = g[f"pcsp0_{M}_data"] if pc else g[f"sp0_{M}_data"]
            assert rel_err(mat.data, ref) <= TOL, M
        rb, rh = (g["pcsp0_b"], g["pcsp0_h"]) if pc else (g["sp0_b"], g["sp0_h"])
        assert rel_err(prog.b, rb) <= TOL and rel_err(prog.h, rh) <= TOL
    assert rel_err(lin.jx, g["ig_jx"]) <= TOL and rel_err(lin.defects, g["ig_defects"]) <= TOL
