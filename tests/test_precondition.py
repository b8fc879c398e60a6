"""Preconditioning of the SCP subproblem on the GPU vs the
reference's `cito.conic.precondition` (/root/reference/pkg/src/cito/conic.py:290-338).

Golden pc{tag}_* arrays were produced by running the UNMODIFIED reference
`precondition` on the reference's own sp0/sp1/sp2 programs
(tests/golden/make_golden_precondition.py).  Row scales and scaled A/G values
are bit-exact (one product per entry, as scipy's Da @ A); b/h scale the GPU's
own b/h (rel <= 1e-9 against the reference's).  The TestPrecondition cases of
the reference (tests/test_conic.py:369-408) are re-expressed on small programs.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_scenario, load_golden, rel_err

CASES = ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]
TAGS = ["sp0", "sp1", "sp2"]


def _program(g, tag):
    from paper_2604_09993_b200.subproblem import ConeSpec, ConicProgram

    n = int(g[f"{tag}_A_shape"][1])
    mat = lambda M: sp.csc_matrix((g[f"{tag}_{M}_data"], g[f"{tag}_{M}_indices"], g[f"{tag}_{M}_indptr"]),  # noqa
                                  shape=tuple(g[f"{tag}_{M}_shape"]))
    P = sp.csc_matrix((g[f"{tag}_P_data"], g[f"{tag}_P_indices"], g[f"{tag}_P_indptr"]), shape=(n, n))
    return ConicProgram(P=P, c=g[f"{tag}_c"], A=mat("A"), b=g[f"{tag}_b"], G=mat("G"), h=g[f"{tag}_h"],
                        cones=ConeSpec(nonneg=int(g[f"{tag}_nonneg"]), soc=tuple(int(d) for d in g[f"{tag}_soc"])))


def _scales_numpy(prog):
    """Test-side restatement of conic.py:290-309 (the checker for the kernels)."""
    def rowmax(M):
        M = sp.csr_matrix(M)
        out = np.zeros(M.shape[0])
        for i in range(M.shape[0]):
            blk = M.data[M.indptr[i]:M.indptr[i + 1]]
            out[i] = np.max(np.abs(blk)) if blk.size else 0.0
        return out

    ra = rowmax(prog.A)
    ra[ra == 0.0] = 1.0
    rg = rowmax(prog.G)
    nn = prog.cones.nonneg
    sg = np.ones(prog.G.shape[0])
    nz = rg[:nn] != 0.0
    sg[:nn][nz] = 1.0 / rg[:nn][nz]
    s0 = nn
    for d in prog.cones.soc:
        m = np.max(rg[s0:s0 + d])
        if m > 0:
            sg[s0:s0 + d] = 1.0 / m
        s0 += d
    return 1.0 / ra, sg


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tag", TAGS)
def test_golden_precondition_restatement(name, tag):
    """CPU: the restated scale rule reproduces the reference's output bit-exactly."""
    g = load_golden(name)
    prog = _program(g, tag)
    sA, sG = _scales_numpy(prog)
    assert np.array_equal(sA, g[f"pc{tag}_row_scale_A"]) and np.array_equal(sG, g[f"pc{tag}_row_scale_G"])
    A = sp.csc_matrix(prog.A)
    assert np.array_equal(sA[A.indices] * A.data, g[f"pc{tag}_A_data"])
    G = sp.csc_matrix(prog.G)
    assert np.array_equal(sG[G.indices] * G.data, g[f"pc{tag}_G_data"])
    assert np.array_equal(sA * prog.b, g[f"pc{tag}_b"]) and np.array_equal(sG * prog.h, g[f"pc{tag}_h"])


def _check_scaled(scaled, prec, g, tag, exact_rhs):
    assert np.array_equal(prec.row_scale_A, g[f"pc{tag}_row_scale_A"])
    assert np.array_equal(prec.row_scale_G, g[f"pc{tag}_row_scale_G"])
    assert prec.cost_scale == float(g[f"pc{tag}_cost_scale"])
    for M in ("A", "G"):
        mat = getattr(scaled, M)
        assert np.array_equal(mat.indptr, g[f"{tag}_{M}_indptr"]) and np.array_equal(mat.indices, g[f"{tag}_{M}_indices"])
        assert np.array_equal(mat.data, g[f"pc{tag}_{M}_data"]), M
    if exact_rhs:
        assert np.array_equal(scaled.b, g[f"pc{tag}_b"]) and np.array_equal(scaled.h, g[f"pc{tag}_h"])
    else:
        assert rel_err(scaled.b, g[f"pc{tag}_b"]) <= 1e-9 and rel_err(scaled.h, g[f"pc{tag}_h"]) <= 1e-9
    assert np.array_equal(scaled.c, g[f"pc{tag}_c"]) and np.array_equal(scaled.P.data, g[f"pc{tag}_P_data"])
    assert np.all(prec.var_scale == 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_precondition_dropin_matches_reference(name, tag):
    """precondition(prog) on a host program (uploaded, scaled by the kernels)."""
    from paper_2604_09993_b200.subproblem import precondition

    g = load_golden(name)
    scaled, prec = precondition(_program(g, tag))
    _check_scaled(scaled, prec, g, tag, exact_rhs=True)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_fused_precondition_matches_reference(name, tag):
    """Assembly with the row norms fused into the CSC write, then scales on the device."""
    import torch

    from paper_2604_09993_b200.scenario import Layout, build_scaling
    from paper_2604_09993_b200.subproblem import LIN_SOURCES, SubproblemAssembler, SubproblemPattern
    from test_subproblem import _lin

    g = load_golden(name)
    sc = golden_scenario(name)
    lay = Layout(sc)
    scale_v, _, _ = build_scaling(sc, lay)
    dev = torch.device("cuda")
    asm = SubproblemAssembler(SubproblemPattern(sc, lay, scale_v), dev)
    lin = _lin(g, tag)
    lin_dev = {k: torch.as_tensor(np.ascontiguousarray(lin[k], dtype=np.float64), device=dev) for k in LIN_SOURCES}
    out = asm.assemble_device(lin_dev, torch.as_tensor(lin["z_ref"], device=dev), precondition=True)
    scaled, prec, meta = asm.to_program(out, g[f"{tag}_zj"])
    _check_scaled(scaled, prec, g, tag, exact_rhs=False)


@pytest.mark.gpu
def test_gpu_build_then_precondition_reuses_device_copy():
    """build_subproblem drop-in followed by the precondition drop-in (scp.py:413-414)."""
    import torch

    from paper_2604_09993_b200.scenario import Layout, build_scaling
    from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern, precondition, _assemblers
    from test_subproblem import _lin
    from paper_2604_09993_b200.subproblem import LIN_SOURCES

    name, tag = "halfcheetah_n30", "sp1"
    g = load_golden(name)
    sc = golden_scenario(name)
    lay = Layout(sc)
    dev = torch.device("cuda")
    asm = SubproblemAssembler(SubproblemPattern(sc, lay, build_scaling(sc, lay)[0]), dev)
    _assemblers[("test", 0)] = asm
    try:
        lin = _lin(g, tag)
        lin_dev = {k: torch.as_tensor(np.ascontiguousarray(lin[k], dtype=np.float64), device=dev) for k in LIN_SOURCES}
        prog, _ = asm.to_program(asm.assemble_device(lin_dev, torch.as_tensor(lin["z_ref"], device=dev)),
                                 g[f"{tag}_zj"])
        assert asm.last[0] is prog
        scaled, prec = precondition(prog)
        _check_scaled(scaled, prec, g, tag, exact_rhs=False)
        # the device path must equal scaling the host copy of the same program
        s2, p2 = precondition(type(prog)(P=prog.P, c=prog.c, A=prog.A.copy(), b=prog.b.copy(), G=prog.G.copy(),
                                         h=prog.h.copy(), cones=prog.cones))
        assert np.array_equal(s2.b, scaled.b) and np.array_equal(s2.G.data, scaled.G.data)
    finally:
        _assemblers.pop(("test", 0), None)


@pytest.mark.gpu
def test_gpu_scp_step_iterate_preconditioned():
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    step = GpuSCPStep(golden_scenario(name))
    lin, scaled, prec, meta = step.iterate(g["ig_z"], 1.0, precondition=True)
    assert np.array_equal(prec.row_scale_G, g["pcsp0_row_scale_G"])
    assert rel_err(prec.row_scale_A, g["pcsp0_row_scale_A"]) <= 1e-9
    for M in ("A", "G"):
        mat = getattr(scaled, M)
        assert np.array_equal(mat.indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(mat.indices, g[f"sp0_{M}_indices"])
        assert rel_err(mat.data, g[f"pcsp0_{M}_data"]) <= 1e-9
    assert rel_err(scaled.b, g["pcsp0_b"]) <= 1e-9 and rel_err(scaled.h, g["pcsp0_h"]) <= 1e-9
    assert abs(prec.cost_scale - float(g["pcsp0_cost_scale"])) <= 1e-12 * float(g["pcsp0_cost_scale"])


def _small(G_rows, h, nonneg, soc=(), A_rows=None, b=None):
    from paper_2604_09993_b200.subproblem import ConeSpec, ConicProgram

    G = sp.csc_matrix(np.asarray(G_rows, dtype=float))
    n = G.shape[1]
    A = sp.csc_matrix(np.asarray(A_rows, dtype=float)) if A_rows is not None else sp.csc_matrix((0, n))
    A.eliminate_zeros()
    G.eliminate_zeros()
    return ConicProgram(P=sp.csc_matrix((n, n)), c=np.zeros(n), A=A, b=np.asarray(b if b is not None else [], float),
                        G=G, h=np.asarray(h, float), cones=ConeSpec(nonneg=nonneg, soc=tuple(soc)))


@pytest.mark.gpu
def test_gpu_precondition_reference_unit_cases():
    """tests/test_conic.py:369-408 (row inf norm, SOC uniform scaling, zero row kept)."""
    from paper_2604_09993_b200.subproblem import precondition

    scaled, prec = precondition(_small([[0.0, 5.0, -10.0]], [2.0], 1))
    assert prec.row_scale_G[0] == pytest.approx(0.1)
    assert np.max(np.abs(scaled.G.toarray()[0])) == pytest.approx(1.0) and scaled.h[0] == pytest.approx(0.2)

    _, prec = precondition(_small([[0.0], [-1.0]], [1.0, 0.0], 2))
    assert prec.row_scale_G[0] == 1.0 and prec.row_scale_G[1] == 1.0

    rows = [[3.0, 0.0], [-1.0, 0.0], [0.0, -40.0], [0.0, 0.5], [2.0, 1.0], [0.0, 0.0], [0.0, 0.0]]
    prog = _small(rows, [1.0, 2.0, 0.0, 0.0, 3.0, 1.0, 0.0], 2, soc=(3, 2),
                  A_rows=[[0.0, 4.0], [0.0, 0.0]], b=[1.0, 0.0])
    scaled, prec = precondition(prog)
    sA, sG = _scales_numpy(prog)
    assert np.array_equal(prec.row_scale_A, sA) and np.array_equal(prec.row_scale_G, sG)
    assert np.all(prec.row_scale_G[2:5] == prec.row_scale_G[2]) and np.all(prec.row_scale_G[5:] == 1.0)
    rng = np.random.default_rng(32)
    for _ in range(20):  # SOC membership preserved (test_conic.py:381-398)
        xv = rng.normal(size=2)
        so, ss = prog.h - prog.G @ xv, scaled.h - scaled.G @ xv
        blk_o, blk_s = so[2:5], ss[2:5]
        assert (blk_o[0] >= np.linalg.norm(blk_o[1:])) == (blk_s[0] >= np.linalg.norm(blk_s[1:]))


@pytest.mark.gpu
def test_gpu_scp_step_graph_replay_equals_eager():
    """GpuSCPStep replays one captured CUDA graph per iteration; delta/epsilon are
    read from device memory, so every delta of the homotopy must give exactly the
    eager result (same kernels, same order)."""
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    sc = golden_scenario(name)
    sg, se = GpuSCPStep(sc, use_graph=True), GpuSCPStep(sc, use_graph=False)
    z = g["ig_z"]
    for delta, pc in ((1.0, False), (0.3, False), (0.05, True), (0.7, True), (0.2, False)):
        rg, re_ = sg.iterate(z, delta, precondition=pc), se.iterate(z, delta, precondition=pc)
        pg, pe = rg[1], re_[1]
        for M in ("A", "G"):
            a, b = getattr(pg, M), getattr(pe, M)
            assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
            assert np.array_equal(a.data, b.data)
        assert np.array_equal(pg.b, pe.b) and np.array_equal(pg.h, pe.h) and np.array_equal(pg.c, pe.c)
        assert np.array_equal(rg[0].psi, re_[0].psi) and np.array_equal(rg[0].theta_jac, re_[0].theta_jac)
    assert sg._plan["graph_kernels"][False] >= 4  # K1, K3, one-pass CSC compaction, rhs
    assert {k for hb in sg._plan["hosts"] for k in hb.graphs} == {False, True}


@pytest.mark.gpu
def test_gpu_scp_step_results_survive_later_iterations():
    """Programs are returned as views of pinned result buffers (no host copy); a
    buffer is reused only when no array of an earlier result is alive."""
    import gc

    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    step = GpuSCPStep(golden_scenario(name))
    _, p1, _ = step.iterate(g["ig_z"], 1.0)
    keep = (p1.A.data.copy(), p1.b.copy(), p1.G.indices.copy())
    z2 = g["ig_z"] + 1e-3 * np.random.default_rng(3).normal(size=g["ig_z"].size)
    for d in (0.5, 0.25, 0.1):
        step.iterate(z2, d)
    assert np.array_equal(p1.A.data, keep[0]) and np.array_equal(p1.b, keep[1])
    assert np.array_equal(p1.G.indices, keep[2])
    n_before = len(step._plan["hosts"])
    del p1
    gc.collect()
    for d in (0.5, 0.25):
        step.iterate(z2, d)
    assert len(step._plan["hosts"]) == n_before  # freed buffers are reused


@pytest.mark.gpu
@pytest.mark.parametrize("precondition", [False, True])
def test_gpu_scp_step_prebuilt_program_rebuilt(precondition):
    """iterate builds the scipy matrices / program over the pinned buffer before the
    synchronisation with the previous call's nonzero counts; a call whose counts
    differ must come back rebuilt and complete (here the prediction is forced
    wrong), and the bytes moved stay below the packed buffer's size."""
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    sc = golden_scenario(name)
    sg, se = GpuSCPStep(sc, use_graph=True), GpuSCPStep(sc, use_graph=False)
    z = g["ig_z"]
    sg.iterate(z, 1.0, precondition=precondition)  # capture
    sg._plan["last_nnz_ag"] = (100, 10)  # pretend the previous call had tiny matrices
    rg = sg.iterate(z, 0.5, precondition=precondition)
    re_ = se.iterate(z, 0.5, precondition=precondition)
    for M in ("A", "G"):
        a, b = getattr(rg[1], M), getattr(re_[1], M)
        assert a.nnz > 100 and np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.data, b.data)
    assert np.array_equal(rg[1].b, re_[1].b) and np.array_equal(rg[1].h, re_[1].h)
    if precondition:
        assert np.array_equal(rg[2].row_scale_A, re_[2].row_scale_A)
    assert sg._plan["last_nnz_ag"] == (rg[1].A.nnz, rg[1].G.nnz)
    assert sg.d2h_bytes(precondition) < sg._plan["pk"].nbytes
