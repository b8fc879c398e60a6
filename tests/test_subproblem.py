"""Full SCP subproblem assembly vs the reference's
build_subproblem -> canonicalize (golden sp0/sp1/sp2: initial guess, perturbed
iterate, nonzero impulses).  CPU: the recipe tables evaluated with numpy
(test-side evaluator) must reproduce the reference CSC bit-exactly; GPU: the
device assembler must match it (indices bit-exact, values rel <= 1e-9)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_scenario, load_golden, rel_err

CASES = ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]
TAGS = ["sp0", "sp1", "sp2"]


def _lin(g, tag):
    node = "nd" if tag == "sp2" else "ig"
    return {"jx": g["ig_jx"], "ju": g["ig_ju"], "js": g["ig_js"], "ends": g["ig_ends"],
            "imp_jac": g[f"{node}_imp_jac"], "theta_jac": g[f"{node}_theta_jac"], "psi_jac": g[f"{node}_psi_jac"],
            "imp_v": g[f"{node}_imp"], "theta": g[f"{node}_theta"], "psi": g[f"{node}_psi"],
            "z_ref": g["nd_z"] if tag == "sp2" else g["ig_z"]}


def _eval_numpy(pat, csc, lin):
    """Test-side evaluator of the recipe tables (mirrors the device kernels)."""
    from paper_2604_09993_b200.subproblem import LIN_SOURCES

    flat = [np.asarray(lin[k], dtype=float).reshape(-1) for k in LIN_SOURCES]
    v = csc["val"].copy()
    m = csc["src"] >= 0
    for s in np.unique(csc["src"][m]):
        sel = m & (csc["src"] == s)
        v[sel] = (csc["val"][sel] * flat[s][csc["idx"][sel]]) * pat.sigma[csc["col"][sel]]
    keep = v != 0.0
    counts = np.bincount(csc["col"][keep], minlength=pat.n)
    indptr = np.concatenate([[0], np.cumsum(counts)])
    return indptr, csc["row"][keep], v[keep]


def _rhs_numpy(pat, csc, rows_desc, lin):
    from paper_2604_09993_b200.subproblem import LIN_SOURCES

    flat = [np.asarray(lin[k], dtype=float).reshape(-1) for k in LIN_SOURCES]
    rhs = csc["rhs"].copy()
    z = lin["z_ref"]
    for row, form, segs, vsrc, voff in rows_desc:
        dot = 0.0
        for s, off, ln, cols in segs:
            dot += flat[s][off:off + ln] @ z[cols]
        val = flat[vsrc][voff]
        rhs[row] = val - dot if form == 0 else dot - val
    return rhs


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tag", TAGS)
def test_recipes_reproduce_reference_csc(name, tag):
    from paper_2604_09993_b200.scenario import Layout, build_scaling
    from paper_2604_09993_b200.subproblem import SubproblemPattern

    g = load_golden(name)
    sc = golden_scenario(name)
    lay = Layout(sc)
    scale_v, _, _ = build_scaling(sc, lay)
    pat = SubproblemPattern(sc, lay, scale_v)
    lin = _lin(g, tag)
    for M, rows in (("A", pat.lin_rows_A), ("G", pat.lin_rows_G)):
        csc = getattr(pat, M)
        indptr, indices, data = _eval_numpy(pat, csc, lin)
        assert tuple(g[f"{tag}_{M}_shape"]) == (csc["nrows"], pat.n)
        assert np.array_equal(indptr, g[f"{tag}_{M}_indptr"]), M
        assert np.array_equal(indices, g[f"{tag}_{M}_indices"]), M
        assert np.array_equal(data, g[f"{tag}_{M}_data"]), M  # identical float ops -> bit-exact
        rhs = _rhs_numpy(pat, csc, rows, lin)
        ref = g[f"{tag}_b"] if M == "A" else g[f"{tag}_h"]
        assert rel_err(rhs, ref) <= 1e-13, M
    assert pat.n_orthant == int(g[f"{tag}_nonneg"]) and pat.soc_dims == tuple(g[f"{tag}_soc"])
    P = sp.csc_matrix((g[f"{tag}_P_data"], g[f"{tag}_P_indices"], g[f"{tag}_P_indptr"]), shape=(pat.n, pat.n))
    assert np.array_equal(P.diagonal(), pat.P_diag) and P.nnz == lay.dim
    assert np.array_equal(pat.objective_c(g[f"{tag}_zj"]), g[f"{tag}_c"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_assembly_matches_reference(name, tag):
    """Device recipe evaluation + zero compaction + rhs == reference canonicalize."""
    import torch

    from paper_2604_09993_b200.scenario import Layout, build_scaling
    from paper_2604_09993_b200.subproblem import LIN_SOURCES, SubproblemAssembler, SubproblemPattern

    g = load_golden(name)
    sc = golden_scenario(name)
    lay = Layout(sc)
    scale_v, _, _ = build_scaling(sc, lay)
    dev = torch.device("cuda")
    asm = SubproblemAssembler(SubproblemPattern(sc, lay, scale_v), dev)
    lin = _lin(g, tag)
    lin_dev = {k: torch.as_tensor(np.ascontiguousarray(lin[k], dtype=np.float64), device=dev) for k in LIN_SOURCES}
    out = asm.assemble_device(lin_dev, torch.as_tensor(lin["z_ref"], device=dev))
    prog, meta = asm.to_program(out, g[f"{tag}_zj"])
    for M in ("A", "G"):
        mat = getattr(prog, M)
        assert np.array_equal(mat.indptr, g[f"{tag}_{M}_indptr"]) and np.array_equal(mat.indices, g[f"{tag}_{M}_indices"])
        assert np.array_equal(mat.data, g[f"{tag}_{M}_data"]), M
    assert rel_err(prog.b, g[f"{tag}_b"]) <= 1e-13 and rel_err(prog.h, g[f"{tag}_h"]) <= 1e-13
    assert np.array_equal(prog.c, g[f"{tag}_c"])
    assert prog.cones.nonneg == int(g[f"{tag}_nonneg"]) and tuple(prog.cones.soc) == tuple(g[f"{tag}_soc"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_linearize_then_assemble_matches_reference(name):
    """Fully device-resident iteration: linearize_all on the GPU, then assembly."""
    import torch

    from paper_2604_09993_b200.linearize import GpuTranscription
    from paper_2604_09993_b200.scenario import build_scaling
    from paper_2604_09993_b200.subproblem import SubproblemAssembler, SubproblemPattern

    g = load_golden(name)
    sc = golden_scenario(name)
    gt = GpuTranscription(sc)
    scale_v, _, _ = build_scaling(sc, gt.lay)
    asm = SubproblemAssembler(SubproblemPattern(sc, gt.lay, scale_v), gt.device)
    z = torch.as_tensor(g["ig_z"], device=gt.device)
    r = gt.linearize_device(z, 1.0)
    out = asm.assemble_device(r, z)
    prog, _ = asm.to_program(out, g["sp0_zj"])
    for M in ("A", "G"):
        mat = getattr(prog, M)
        assert np.array_equal(mat.indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(mat.indices, g[f"sp0_{M}_indices"])
        assert rel_err(mat.data, g[f"sp0_{M}_data"]) <= 1e-9, M
    assert rel_err(prog.b, g["sp0_b"]) <= 1e-9 and rel_err(prog.h, g["sp0_h"]) <= 1e-9


@pytest.mark.gpu
def test_gpu_scp_step_iterate_matches_reference():
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    step = GpuSCPStep(golden_scenario(name))
    lin, prog, meta = step.iterate(g["ig_z"], 1.0)
    for M in ("A", "G"):
        mat = getattr(prog, M)
        assert np.array_equal(mat.indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(mat.indices, g[f"sp0_{M}_indices"])
        assert rel_err(mat.data, g[f"sp0_{M}_data"]) <= 1e-9
    assert rel_err(lin.jx, g["ig_jx"]) <= 1e-9 and rel_err(lin.defects, g["ig_defects"]) <= 1e-9
    with pytest.raises(FloatingPointError):
        step.iterate(np.full_like(g["ig_z"], np.nan), 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_scp_step_all_models_match_reference(name):
    """GpuSCPStep (captured graph, packed result) on every golden model: pattern
    bit-exact and values rel <= 1e-9 against the reference's build_subproblem."""
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    g = load_golden(name)
    step = GpuSCPStep(golden_scenario(name))
    for _ in range(2):  # first call captures the graph, second replays it
        lin, prog, meta = step.iterate(g["ig_z"], 1.0, z_j=g["sp0_zj"])
        for M in ("A", "G"):
            mat = getattr(prog, M)
            assert np.array_equal(mat.indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(mat.indices,
                                                                                      g[f"sp0_{M}_indices"])
            assert rel_err(mat.data, g[f"sp0_{M}_data"]) <= 1e-9, M
        assert rel_err(prog.b, g["sp0_b"]) <= 1e-9 and rel_err(prog.h, g["sp0_h"]) <= 1e-9
        assert np.array_equal(prog.c, g["sp0_c"])


def test_csc_direct_equals_scipy_constructor():
    """GpuSCPStep's direct csc_matrix construction (no per-call constructor checks)
    gives the same matrix object state as scipy's constructor and a valid format."""
    import paper_2604_09993_b200.subproblem as SPB
    from paper_2604_09993_b200.subproblem import _csc_direct

    SPB._CSC_FAST = None  # probe again: this test must see the probe call first
    A = sp.random(40, 70, density=0.15, format="csc", random_state=3)
    A.sort_indices()
    d, i, p = A.data.copy(), A.indices.astype(np.int32), A.indptr.astype(np.int32)
    first = _csc_direct(d, i, p, A.shape)  # the probe (regular constructor)
    fast = _csc_direct(d, i, p, A.shape)
    assert set(vars(fast)) == set(vars(first))  # before any lazily cached attribute
    assert fast.data is d and fast.indices is i and fast.indptr is p  # no copies
    for m in (first, fast):
        assert isinstance(m, sp.csc_matrix) and m.shape == A.shape
        m.check_format(full_check=True)
        assert (m != A).nnz == 0 and m.has_sorted_indices
        assert np.array_equal(m.toarray(), A.toarray()) and np.allclose(m.T @ np.ones(40), A.T @ np.ones(40))


def test_csc_direct_rejects_inconsistent_arrays():
    from paper_2604_09993_b200.subproblem import _csc_direct

    d, i = np.ones(3), np.array([0, 1, 2], dtype=np.int32)
    with pytest.raises(RuntimeError):
        _csc_direct(d, i, np.array([0, 1, 4], dtype=np.int32), (3, 2))  # indptr[-1] != nnz
    with pytest.raises(RuntimeError):
        _csc_direct(d, i, np.array([1, 2, 3], dtype=np.int32), (3, 2))  # indptr[0] != 0
    with pytest.raises(RuntimeError):
        _csc_direct(d, i.astype(np.int64), np.array([0, 1, 3], dtype=np.int32), (3, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pointmass_rest", "halfcheetah_n30"])
@pytest.mark.parametrize("precondition", [False, True])
def test_gpu_scp_step_graph_replay_pattern_change(name, precondition):
    """A captured iteration replayed at a point whose pattern differs (nonzero
    impulses) must equal a fresh step at that point bit for bit: more nonzeros
    than the captured call, the pattern stamp, the row indices fetched after the
    synchronisation, the program objects rebuilt for the new counts."""
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    g = load_golden(name)
    sc = golden_scenario(name)
    lay_dim = g["ig_z"].size
    rng = np.random.default_rng(3)
    z2 = g["ig_z"].copy()
    from paper_2604_09993_b200.scenario import Layout

    lay = Layout(sc)
    for k in range(lay.N):  # impulses on: more nonzeros in the node rows
        z2[lay.phi(k)] = rng.uniform(0.1, 0.5, size=2 * lay.n_c)
    assert z2.size == lay_dim
    a = GpuSCPStep(sc)
    for _ in range(2):
        a.iterate(g["ig_z"], 1.0, precondition=precondition)
    ra = a.iterate(z2, 0.5, precondition=precondition)
    rb = GpuSCPStep(sc, use_graph=False).iterate(z2, 0.5, precondition=precondition)
    for M in ("A", "G"):
        ma, mb = getattr(ra[1], M), getattr(rb[1], M)
        assert np.array_equal(ma.indptr, mb.indptr) and np.array_equal(ma.indices, mb.indices)
        assert np.array_equal(ma.data, mb.data)
    assert np.array_equal(ra[1].b, rb[1].b) and np.array_equal(ra[1].h, rb[1].h)
    ra2 = a.iterate(g["ig_z"], 1.0, precondition=precondition)  # and back
    rc = GpuSCPStep(sc, use_graph=False).iterate(g["ig_z"], 1.0, precondition=precondition)
    assert np.array_equal(ra2[1].A.data, rc[1].A.data) and np.array_equal(ra2[1].A.indices, rc[1].A.indices)


@pytest.mark.gpu
@pytest.mark.parametrize("precondition", [False, True])
def test_gpu_scp_step_pattern_stamp_sequence(precondition):
    """The CSC row indices come back only into a result buffer that does not hold
    the current pattern (the compaction stamps a moved pattern): a sequence of
    points whose patterns alternate, with the previous result kept alive like
    cito.scp.solve and sometimes dropped, must give every program bit-equal to a
    fresh eager step at the same point."""
    from paper_2604_09993_b200.scenario import Layout
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    sc = golden_scenario(name)
    lay = Layout(sc)
    rng = np.random.default_rng(5)
    z1 = g["ig_z"]
    z2 = z1.copy()
    for k in range(lay.N):  # impulses on: a different pattern
        z2[lay.phi(k)] = rng.uniform(0.1, 0.5, size=2 * lay.n_c)
    pts = {"1": (z1, 0.7), "2": (z2, 0.7), "3": (z2, 0.4)}
    ref = {k: GpuSCPStep(sc, use_graph=False).iterate(z, d, precondition=precondition)[1] for k, (z, d) in pts.items()}
    pat = lambda p: [getattr(p, M).indptr for M in ("A", "G")] + [getattr(p, M).indices for M in ("A", "G")]  # noqa
    assert not all(np.array_equal(u, v) for u, v in zip(pat(ref["1"]), pat(ref["2"])))
    step = GpuSCPStep(sc)
    keep = None
    seq = ["1", "2", "2", "1", "1", "3", "2", "1", "1", "1", "3", "3"]
    for i, key in enumerate(seq):
        r = step.iterate(*pts[key], precondition=precondition)
        prog = r[1]
        for M in ("A", "G"):
            ma, mb = getattr(prog, M), getattr(ref[key], M)
            assert np.array_equal(ma.indptr, mb.indptr) and np.array_equal(ma.indices, mb.indices), (i, key, M)
            assert np.array_equal(ma.data, mb.data), (i, key, M)
        assert np.array_equal(prog.b, ref[key].b) and np.array_equal(prog.h, ref[key].h)
        keep = r if i % 4 != 3 else None  # hold the previous result (two buffers in use) most of the time
        del r, prog
    assert len(step._plan["hosts"]) >= 2
    assert step.pattern_refetches > 0  # a pattern moved under a buffer that held the previous one
    # steady state (same pattern, buffer up to date): values only
    b0 = step.d2h_copied
    r = step.iterate(*pts["3"], precondition=precondition)
    r = step.iterate(*pts["3"], precondition=precondition)
    b1 = step.d2h_copied
    r = step.iterate(*pts["3"], precondition=precondition)
    assert step.d2h_copied - b1 == step.d2h_bytes(precondition) and b1 > b0
    assert step.d2h_bytes(precondition) < step.d2h_bytes(precondition, indices=True)


@pytest.mark.gpu
def test_gpu_scp_step_mixed_modes_same_buffer():
    """Plain and preconditioned calls alternating on the same result buffer: the
    constant b/h rows live in the host buffer (scaled there by a preconditioned
    call and restored before a plain one), so every program must equal a fresh
    step of its own mode."""
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    sc = golden_scenario(name)
    z = g["ig_z"]
    ref = {pc: GpuSCPStep(sc, use_graph=False).iterate(z, 0.8, precondition=pc)[1] for pc in (False, True)}
    step = GpuSCPStep(sc)
    for pc in (False, True, False, False, True, True, False):
        prog = step.iterate(z, 0.8, precondition=pc)[1]
        assert np.array_equal(prog.b, ref[pc].b) and np.array_equal(prog.h, ref[pc].h), pc
        assert np.array_equal(prog.A.data, ref[pc].A.data) and np.array_equal(prog.G.data, ref[pc].G.data), pc
        del prog  # the next call reuses a buffer (the last preconditioned one stays held for unscaled_program)
    assert len(step._plan["hosts"]) <= 2


@pytest.mark.gpu
def test_gpu_scp_step_reserve_keeps_live_results():
    """reserve() captures graphs by running an iteration into result buffers: it must
    not write into a buffer a live result points into."""
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    sc = golden_scenario(name)
    step = GpuSCPStep(sc)
    live = step.iterate(g["ig_z"], 1.0)[1]  # plain result, held
    saved = [live.A.data.copy(), live.b.copy(), live.G.data.copy()]
    step.reserve(2, precondition=True)  # preconditioned graphs: would scale a live buffer
    assert np.array_equal(live.A.data, saved[0]) and np.array_equal(live.b, saved[1])
    assert np.array_equal(live.G.data, saved[2])
    assert sum(1 for hb in step._plan["hosts"] if True in hb.graphs) >= 2


@pytest.mark.gpu
def test_gpu_scp_step_results_outlive_the_step():
    """The program's arrays live in the step's pinned result buffer; they keep that
    allocation alive after the GpuSCPStep itself is dropped."""
    import gc

    from paper_2604_09993_b200.subproblem import GpuSCPStep

    name = "halfcheetah_n30"
    g = load_golden(name)
    sc = golden_scenario(name)
    prog = GpuSCPStep(sc).iterate(g["ig_z"], 1.0)[1]
    saved = [a.copy() for a in (prog.A.data, prog.A.indices, prog.G.data, prog.b)]
    gc.collect()
    for _ in range(3):  # other steps allocate (and fill) pinned buffers of the same size
        GpuSCPStep(sc).iterate(g["ig_z"] * 0.5, 0.3)
    for a, b in zip((prog.A.data, prog.A.indices, prog.G.data, prog.b), saved):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name", CASES)
def test_packed_records_reproduce_reference_csc(name):
    """The 16-byte records of k_csc_flat (subproblem.packed_entries), evaluated on the
    host exactly as the kernel does (lin * w with w = sign * sigma folded), give the
    reference CSC bit for bit; the tile column table covers every column once."""
    from paper_2604_09993_b200.scenario import Layout, build_scaling
    from paper_2604_09993_b200.subproblem import LIN_SOURCES, SubproblemPattern, packed_entries

    g = load_golden(name)
    sc = golden_scenario(name)
    lay = Layout(sc)
    pat = SubproblemPattern(sc, lay, build_scaling(sc, lay)[0])
    lin = _lin(g, "sp0")
    flat = [np.asarray(lin[k], dtype=float).reshape(-1) for k in LIN_SOURCES]
    for M in ("A", "G"):
        csc = getattr(pat, M)
        rec, tcol = packed_entries(csc, pat.sigma_full())
        src = (rec["key"] >> 27).astype(np.int64) - 1
        idx = (rec["key"] & ((1 << 27) - 1)).astype(np.int64)
        v = rec["w"].copy()
        for s in np.unique(src[src >= 0]):
            sel = src == s
            v[sel] = flat[s][idx[sel]] * rec["w"][sel]
        keep = v != 0.0
        indptr = np.concatenate([[0], np.cumsum(np.bincount(csc["col"][keep], minlength=pat.n))])
        assert np.array_equal(indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(rec["row"][keep], g[f"sp0_{M}_indices"])
        assert np.array_equal(v[keep], g[f"sp0_{M}_data"]), M
        ntile = len(tcol) - 1
        assert ntile == max(1, -(-rec.size // 2048)) and tcol[0] == 0 and tcol[-1] == pat.n + 1
        sp = csc["indptr"]
        for t in range(ntile):  # columns owned by tile t start inside it (the last tile takes the tail)
            cols = np.arange(tcol[t], min(tcol[t + 1], pat.n + 1))
            assert np.all(sp[cols] >= 2048 * t)
            if t < ntile - 1:
                assert np.all(sp[cols] < 2048 * (t + 1))
