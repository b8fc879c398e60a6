"""CSC scatter of the multiple-shooting rows (K4) vs the reference's own
build_subproblem -> canonicalize output (golden, tests/golden/make_golden.py).
Pattern/indices must be bit-exact; values rel <= 1e-9."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_scenario, load_golden, rel_err

CASES = ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]


def _ref_dyn(g, lay):
    # csc_* (make_golden.py) and sp0_* (make_golden_subproblem.py) are the same reference
    # build_subproblem call (initial guess, delta = 1); biped_walk carries only sp0_*
    t = "csc" if "csc_A_data" in g else "sp0"
    A = sp.csc_matrix((g[f"{t}_A_data"], g[f"{t}_A_indices"], g[f"{t}_A_indptr"]), shape=tuple(g[f"{t}_A_shape"]))
    n_dyn = (lay.N - 1) * lay.n_xt
    Ad = A[:n_dyn, :].tocsc()
    Ad.sort_indices()
    return A, Ad, n_dyn


@pytest.mark.parametrize("name", CASES)
def test_pattern_matches_reference_csc(name):
    from paper_2604_09993_b200.scatter import DynamicsCSC, n_cols
    from paper_2604_09993_b200.scenario import Layout, build_scaling

    g = load_golden(name)
    sc = golden_scenario(name)
    lay = Layout(sc)
    A, Ad, n_dyn = _ref_dyn(g, lay)
    n_psi = 3 * lay.n_c + lay.n_g_out
    assert n_cols(lay, n_psi) == A.shape[1]
    _, state_scale, _ = build_scaling(sc, lay)
    pat = DynamicsCSC(lay, A.shape[1], state_scale, g["ig_jx"] != 0, g["ig_ju"] != 0, g["ig_js"] != 0)
    assert np.array_equal(pat.indptr, Ad.indptr.astype(np.int32))
    assert np.array_equal(pat.indices, Ad.indices.astype(np.int32))
    # constant entries carry exactly the reference values
    data = pat.template_data()
    assert np.array_equal(data[pat.const_pos], Ad.data[pat.const_pos])
    # slots into the full reference A agree with the pattern's own ordering
    sx, su, ss = DynamicsCSC.slots_into(A.indptr, A.indices, lay)
    assert ((sx >= 0) == pat.slot_x.__ge__(0)).all() and ((su >= 0) == (pat.slot_u >= 0)).all()
    # host restatement of the values, exactly as scp.py:186-201 computes them
    _, sx_, su_ = build_scaling(sc, lay)
    vx = -g["ig_jx"] * state_scale[None, None, :]
    assert np.array_equal(A.data[sx[sx >= 0]], vx[sx >= 0])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_scatter_values_match_reference(name):
    import torch

    from paper_2604_09993_b200.linearize import GpuTranscription
    from paper_2604_09993_b200.scatter import DynamicsCSC, DynamicsScatter
    from paper_2604_09993_b200.scenario import Layout, build_scaling

    g = load_golden(name)
    sc = golden_scenario(name)
    gt = GpuTranscription(sc)
    lay = gt.lay
    A, Ad, n_dyn = _ref_dyn(g, lay)
    scale_v, state_scale, u_scale = build_scaling(sc, lay)
    dev = gt.device
    z = torch.as_tensor(g["ig_z"], device=dev)
    r = gt.linearize_device(z, float(g["ig_delta"]))
    scat = DynamicsScatter(gt.disc, lay, state_scale, u_scale, sc.s_nominal, dev)
    pat = scat.build_pattern(r["jx"].cpu().numpy(), r["ju"].cpu().numpy(), r["js"].cpu().numpy(), A.shape[1],
                             state_scale)
    assert np.array_equal(pat.indices, Ad.indices) and np.array_equal(pat.indptr, Ad.indptr)
    data = torch.as_tensor(pat.template_data(), device=dev)
    b = torch.empty(n_dyn, dtype=torch.float64, device=dev)
    mm = scat.scatter(r["ends"], r["jx"], r["ju"], r["js"], z, data, b)
    torch.cuda.synchronize()
    assert int(mm.item()) == 0
    assert rel_err(data.cpu().numpy(), Ad.data) <= 1e-9
    assert rel_err(b.cpu().numpy(), g["csc_b" if "csc_b" in g else "sp0_b"][:n_dyn]) <= 1e-9
    # and straight into the reference's full A.data (other rows untouched)
    sx, su, ss = DynamicsCSC.slots_into(A.indptr, A.indices, lay)
    scat.set_slots(sx, su, ss)
    full = torch.as_tensor(A.data.copy(), device=dev)
    keep = full.clone()
    mm = scat.scatter(r["ends"], r["jx"], r["ju"], r["js"], z, full, b)
    torch.cuda.synchronize()
    assert int(mm.item()) == 0
    assert rel_err(full.cpu().numpy(), A.data) <= 1e-9
    touched = np.zeros(A.data.size, bool)
    for s_ in (sx, su, ss):
        touched[s_[s_ >= 0]] = True
    assert np.array_equal(full.cpu().numpy()[~touched], keep.cpu().numpy()[~touched])


@pytest.mark.gpu
def test_linearize_all_matches_reference_golden():
    """GpuTranscription.linearize_all == cito.scp.linearize_all at the initial guess."""
    from paper_2604_09993_b200.linearize import GpuTranscription

    for name in ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]:
        g = load_golden(name)
        gt = GpuTranscription(golden_scenario(name))
        lin = gt.linearize_all(g["ig_z"], float(g["ig_delta"]))
        for f, k in (("ends", "ig_ends"), ("jx", "ig_jx"), ("ju", "ig_ju"), ("js", "ig_js"),
                     ("defects", "ig_defects"), ("psi", "ig_psi"), ("psi_jac", "ig_psi_jac"),
                     ("theta", "ig_theta"), ("theta_jac", "ig_theta_jac"), ("imp_v", "ig_imp"),
                     ("imp_jac", "ig_imp_jac")):
            assert rel_err(getattr(lin, f), g[k]) <= 1e-9, (name, f)
        with pytest.raises(FloatingPointError):
            gt.linearize_all(np.full_like(g["ig_z"], np.nan), 1.0)


@pytest.mark.gpu
def test_linearize_all_exact_zero_pattern_equals_reference():
    """The subproblem CSC drops exact zeros (conic.py:99-125), so every Jacobian entry
    that is an exact zero in the reference must be one here and vice versa -- including
    rounding residues of mathematically-zero entries (the node kernel's elimination order)."""
    from paper_2604_09993_b200.linearize import GpuTranscription

    for name in ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]:
        g = load_golden(name)
        gt = GpuTranscription(golden_scenario(name))
        lin = gt.linearize_all(g["ig_z"], float(g["ig_delta"]))
        for f, k in (("jx", "ig_jx"), ("ju", "ig_ju"), ("js", "ig_js"), ("psi_jac", "ig_psi_jac"),
                     ("theta_jac", "ig_theta_jac"), ("imp_jac", "ig_imp_jac")):
            assert np.array_equal(getattr(lin, f) == 0, g[k] == 0), (name, f)


@pytest.mark.gpu
def test_node_relations_random_z_vs_reference():
    import torch

    from paper_2604_09993_b200.linearize import GpuTranscription, node_inputs

    for name in ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]:
        g = load_golden(name)
        gt = GpuTranscription(golden_scenario(name))
        yp, tv = node_inputs(gt.lay, g["nd_z"])
        out = gt.nodes.host(yp, tv, float(g["nd_delta"]), gt.scenario.ctcs_epsilon)
        for a, k in zip(out, ("psi", "psi_jac", "theta", "theta_jac", "imp", "imp_jac")):
            assert rel_err(a, g["nd_" + k]) <= 1e-9, (name, k)


@pytest.mark.gpu
def test_multistart_batch_equals_single_problems():
    """n_problems > 1 in cito_linearize_all_dev == one call per problem (configs[3] path)."""
    import torch

    from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess

    sc = golden_scenario("halfcheetah_n30")
    gt = GpuTranscription(sc)
    Z = np.stack([initial_guess(sc, gt.disc, gt.lay, seed=s) for s in range(3)])
    Z[1] += 0.01 * np.random.default_rng(0).normal(size=Z.shape[1])
    zd = torch.as_tensor(Z, device=gt.device)
    allp = gt.linearize_device(zd, 0.5)
    n_int, n_node = gt.lay.N - 1, gt.lay.N
    for p in range(3):
        one = gt.linearize_device(zd[p].contiguous(), 0.5)
        for k, v in one.items():
            rows = n_node if k in ("theta", "theta_jac", "imp_v", "imp_jac") else n_int
            got = allp[k][p * rows:(p + 1) * rows]
            assert rel_err(got.cpu().numpy(), v.cpu().numpy()) <= 1e-12, k


@pytest.mark.gpu
def test_linearize_to_host_chunked_equals_device():
    """GpuTranscription.linearize_to_host (multi-start, host arrays, chunked D2H pipeline)
    == one linearize_device call over all problems; fresh and caller-owned outputs."""
    import torch

    from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess_batch

    sc = golden_scenario("halfcheetah_n30")
    gt = GpuTranscription(sc)
    per = (3 * torch.cuda.get_device_properties(0).multi_processor_count) // (gt.lay.N - 1)
    P = 2 * per + 3  # two chunks, the last one taking the remainder
    Z = initial_guess_batch(sc, gt.disc, list(range(P)), gt.lay)
    ref = {k: v.cpu().numpy() for k, v in gt.linearize_device(torch.as_tensor(Z, device=gt.device), 0.5).items()}
    got = gt.linearize_to_host(Z, 0.5)
    pinned = {k: torch.empty(v.shape, dtype=torch.int32 if v.dtype == np.int32 else torch.float64,
                             pin_memory=True).numpy() for k, v in ref.items()}
    got2 = gt.linearize_to_host(torch.as_tensor(Z).pin_memory(), 0.5, out=pinned)
    assert got2 is pinned
    for k, v in ref.items():
        assert np.array_equal(got[k], v) and np.array_equal(pinned[k], v), k
    Z[P - 1, :] = np.nan
    with pytest.raises(FloatingPointError):
        gt.linearize_to_host(Z, 0.5)


@pytest.mark.gpu
def test_initial_guess_matches_reference_and_batch():
    """GPU initial guess == the reference's initial_guess (golden ig_z); the
    multi-start batched version == one call per seed."""
    from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess, initial_guess_batch

    for name in ["pointmass_rest", "monoped_n20", "halfcheetah_n30"]:
        g = load_golden(name)
        sc = golden_scenario(name)
        gt = GpuTranscription(sc)
        z = initial_guess(sc, gt.disc, gt.lay)
        assert rel_err(z, g["ig_z"]) <= 1e-9, name
        Z = initial_guess_batch(sc, gt.disc, [sc.seed, 3, 11], gt.lay)
        assert np.array_equal(Z[0], z)
        assert np.array_equal(Z[2], initial_guess(sc, gt.disc, gt.lay, seed=11))


@pytest.mark.gpu
@pytest.mark.parametrize("P", [6, 12])
def test_multistart_on_batch_kernels_equals_single_problems(P):
    """Multi-start batches large enough for the lockstep batch kernels (6 x 29 = 174
    intervals: 2 per CTA; 12 x 29 = 348: 3 per CTA) read z in-kernel exactly like
    the single-problem latency kernel."""
    import torch

    from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess_batch

    sc = golden_scenario("halfcheetah_n30")
    gt = GpuTranscription(sc)
    Z = initial_guess_batch(sc, gt.disc, list(range(P)), gt.lay)
    zd = torch.as_tensor(Z, device=gt.device)
    allp = gt.linearize_device(zd, 0.3)
    n_int, n_node = gt.lay.N - 1, gt.lay.N
    for p in (0, P // 2, P - 1):
        one = gt.linearize_device(zd[p].contiguous(), 0.3)
        for k, v in one.items():
            rows = n_node if k in ("theta", "theta_jac", "imp_v", "imp_jac") else n_int
            got = allp[k][p * rows:(p + 1) * rows]
            assert rel_err(got.cpu().numpy(), v.cpu().numpy()) <= 1e-11, (P, k)
