"""GPU parity of the discretize/linearize path (K1/K2) through the C ABI.

Checked against (a) golden vectors from the unmodified reference, (b) the C
oracle on larger seeded batches, (c) the reference's own hot-path tests
re-expressed (tests/test_augmentation.py, tests/test_acceptance.py).
Tolerance: rel <= 1e-9 (north star), measured as the reference's _rel_err.
"""

import threading

import numpy as np
import pytest

import pyoracle
from conftest import golden_scenario, load_golden, rel_err, scenario_desc

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _disc(sc):
    from paper_2604_09993_b200 import Discretizer

    g, n_g = sc.path_constraints()
    return Discretizer(sc.model, mixing=sc.mixing_matrix(n_g), path_fn=g, substeps=sc.substeps)


def _ig_batch(sc, z):
    from paper_2604_09993_b200.scenario import Layout

    lay = Layout(sc)
    starts = np.stack([z[lay.xp(k)] for k in range(lay.N - 1)])
    Us = np.stack([z[lay.u(k)] for k in range(lay.N - 1)])
    Ss = np.array([z[lay.s(k)][0] for k in range(lay.N - 1)])
    return starts, Us, Ss


def test_linearize_vs_reference_golden(golden_case):
    name, g, sc = golden_case
    disc = _disc(sc)
    e, jx, ju, js = disc.linearize_batch(g["lin_xt0"], g["lin_U"], g["lin_S"])
    for a, k in ((e, "lin_ends"), (jx, "lin_jx"), (ju, "lin_ju"), (js, "lin_js")):
        assert rel_err(a, g[k]) <= TOL, (name, k, rel_err(a, g[k]))
    starts, Us, Ss = _ig_batch(sc, g["ig_z"])
    e, jx, ju, js = disc.linearize_batch(starts, Us, Ss)
    for a, k in ((e, "ig_ends"), (jx, "ig_jx"), (ju, "ig_ju"), (js, "ig_js")):
        assert rel_err(a, g[k]) <= TOL, (name, k, rel_err(a, g[k]))
        if k != "ig_ends":  # CSC pattern parity needs the exact-zero pattern (cito/scp.py:190-191)
            assert np.array_equal(a != 0.0, g[k] != 0.0), (name, k)


@pytest.mark.parametrize("name,B", [("halfcheetah_n30", 512), ("monoped_n20", 512), ("biped_walk", 96),
                                    ("pointmass_rest", 256)])
def test_linearize_vs_oracle_batch(name, B):
    from paper_2604_09993_b200 import synth

    sc = golden_scenario(name)
    desc = scenario_desc(sc)
    xt0, U, S, _ = synth.random_intervals(sc, B, seed=11, finite_fn=lambda x, u, s: synth.well_posed(
        pyoracle.propagate(desc, sc.substeps, x, u, s)[0]))
    e0, jx0, ju0, js0, bad = pyoracle.linearize(desc, sc.substeps, xt0, U, S)
    e, jx, ju, js = _disc(sc).linearize_batch(xt0, U, S)
    worst = 0.0
    for b in range(B):  # per interval, so a single bad interval cannot hide behind the batch max
        for a, r in ((e, e0), (jx, jx0), (ju, ju0), (js, js0)):
            worst = max(worst, rel_err(a[b], r[b]))
    assert worst <= TOL, (name, worst)


def test_propagate_matches_linearize_and_oracle():
    from paper_2604_09993_b200 import synth

    sc = golden_scenario("halfcheetah_n30")
    desc = scenario_desc(sc)
    xt0, U, S = synth.random_intervals(sc, 300, seed=3)
    ok = pyoracle.propagate(desc, sc.substeps, xt0, U, S)[1] == 0
    xt0, U, S = xt0[ok], U[ok], S[ok]
    disc = _disc(sc)
    ends = disc.propagate_batch(xt0, U, S)
    e0, _ = pyoracle.propagate(desc, sc.substeps, xt0, U, S)
    assert rel_err(ends, e0) <= TOL
    e1, *_ = disc.linearize_batch(xt0, U, S)
    assert rel_err(ends, e1) <= 1e-13
    one = disc.propagate(xt0[0], U[0].reshape(2, -1), float(S[0]))
    assert one.shape == (disc.n_xt,) and rel_err(one, ends[0]) <= 1e-13


def test_nonfinite_raises():
    """tests/test_augmentation.py:201-205 and augmentation.py:231-233 semantics."""
    from paper_2604_09993_b200 import Discretizer
    from paper_2604_09993_b200.model import build_path_constraints
    from test_reference_models import point_mass_model

    m = point_mass_model()
    disc = Discretizer(m)
    with pytest.raises(FloatingPointError):
        disc.propagate(np.full(disc.n_xt, np.nan), np.zeros((2, 3)), 1.0)
    xs = np.zeros((3, disc.n_xt))
    xs[1, 0] = np.nan
    with pytest.raises(FloatingPointError, match=r"\[1\]"):
        disc.propagate_batch(xs, np.zeros((3, 6)), [0.1, 0.1, 0.1])
    with pytest.raises(FloatingPointError):
        disc.linearize_batch(xs, np.zeros((3, 6)), [0.1, 0.1, 0.1])
    g, n_g = build_path_constraints(m)
    with pytest.raises(ValueError):
        Discretizer(m, np.eye(n_g), g, substeps=0)


def test_threaded_calls_equal_serial():
    """linearize_all(jobs>1) fans out over threads (scp.py:101-112); equality to 1e-12
    (tests/test_cli.py:221-230)."""
    from paper_2604_09993_b200 import synth

    sc = golden_scenario("monoped_n20")
    disc = _disc(sc)
    xt0, U, S = synth.random_intervals(sc, 64, seed=5)
    ref = disc.linearize_batch(xt0, U, S)
    bounds = np.linspace(0, 64, 5).astype(int)
    parts = [None] * 4

    def work(i):
        a, b = bounds[i], bounds[i + 1]
        parts[i] = disc.linearize_batch(xt0[a:b], U[a:b], S[a:b])

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for j in range(4):
        cat = np.concatenate([p[j] for p in parts])
        assert np.max(np.abs(cat - ref[j])) <= 1e-12


def test_device_path_matches_host_path():
    import torch

    from paper_2604_09993_b200 import synth

    sc = golden_scenario("halfcheetah_n30")
    disc = _disc(sc)
    xt0, U, S = synth.random_intervals(sc, 64, seed=2)
    host = disc.linearize_batch(xt0, U, S)
    dev = torch.device("cuda")
    out = disc.linearize_batch_device(torch.as_tensor(xt0, device=dev), torch.as_tensor(U, device=dev),
                                      torch.as_tensor(S, device=dev))
    torch.cuda.synchronize()
    for a, b in zip(host, out[:4]):
        assert np.array_equal(a, b.cpu().numpy())
    assert disc.launch_count() >= 2


def test_chunked_host_pipeline_matches_device_path():
    """Batches of >= 4 waves go through the chunked D2H pipeline of cito_linearize_host
    (one-wave chunks, the last one taking the remainder): same bits as one device launch,
    into fresh arrays and into caller-owned (page-locked) out= buffers."""
    import torch

    from paper_2604_09993_b200 import synth

    sc = golden_scenario("halfcheetah_n30")
    disc = _disc(sc)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    B = 4 * 3 * n_sm + 37
    xt0, U, S = synth.random_intervals(sc, B, seed=5)
    n0 = disc.launch_count()
    host = disc.linearize_batch(xt0, U, S)
    assert disc.launch_count() - n0 == 4  # four chunks
    dev = torch.device("cuda")
    out = disc.linearize_batch_device(torch.as_tensor(xt0, device=dev), torch.as_tensor(U, device=dev),
                                      torch.as_tensor(S, device=dev))
    torch.cuda.synchronize()
    for a, b in zip(host, out[:4]):
        assert np.array_equal(a, b.cpu().numpy())
    pinned = tuple(torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy() for a in host)
    res = disc.linearize_batch(xt0, U, S, out=pinned)
    for a, b, r in zip(host, pinned, res):
        assert r is b and np.array_equal(a, b)
    with pytest.raises(ValueError):
        disc.linearize_batch(xt0, U, S, out=(pinned[0], pinned[1], pinned[2], pinned[3][:-1]))


@pytest.mark.parametrize("substeps,B", [(1, 40), (8, 199), (10, 64), (8, 600)])
def test_linearize_substeps_vs_oracle(substeps, B):
    """Other substep counts (configs[4]: 8 substeps, N=200 -> 199 intervals) on both K1
    generations (B <= #SMs: the latency kernel; B > #SMs: the batch kernel)."""
    from dataclasses import replace

    from paper_2604_09993_b200 import synth

    sc = replace(golden_scenario("halfcheetah_n30"), substeps=substeps)
    desc = scenario_desc(sc)
    xt0, U, S, _ = synth.random_intervals(sc, B, seed=substeps, finite_fn=lambda x, u, s: synth.well_posed(
        pyoracle.propagate(desc, sc.substeps, x, u, s)[0]))
    e0, jx0, ju0, js0, _ = pyoracle.linearize(desc, sc.substeps, xt0, U, S)
    e, jx, ju, js = _disc(sc).linearize_batch(xt0, U, S)
    worst = max(rel_err(a[b], r[b]) for b in range(B) for a, r in ((e, e0), (jx, jx0), (ju, ju0), (js, js0)))
    assert worst <= TOL, worst
    ends = _disc(sc).propagate_batch(xt0, U, S)
    assert rel_err(ends, e0) <= TOL


def test_linearize_empty_batch():
    sc = golden_scenario("monoped_n20")
    d = _disc(sc)
    e, jx, ju, js = d.linearize_batch(np.zeros((0, d.n_xt)), np.zeros((0, 2 * d.n_u)), np.zeros(0))
    assert e.shape == (0, d.n_xt) and jx.shape == (0, d.n_xt, d.n_xt) and ju.shape == (0, d.n_xt, 2 * d.n_u)
    assert d.propagate_batch(np.zeros((0, d.n_xt)), np.zeros((0, 2 * d.n_u)), np.zeros(0)).shape == (0, d.n_xt)


def test_linearize_configs2_batch_4096_vs_oracle():
    """configs[2] at its bench size: 4096 synthetic HalfCheetah intervals in one device
    launch (the 3-interval lockstep batch kernel) and through the chunked host pipeline,
    every interval against the oracle (rel <= 1e-9) with the oracle's exact-zero pattern."""
    import torch

    from paper_2604_09993_b200 import synth

    sc = golden_scenario("halfcheetah_n30")
    desc = scenario_desc(sc)
    B = 4096
    xt0, U, S, _ = synth.random_intervals(sc, B, seed=100, finite_fn=lambda x, u, s: synth.well_posed(
        pyoracle.propagate(desc, sc.substeps, x, u, s)[0]))
    ref = pyoracle.linearize(desc, sc.substeps, xt0, U, S)[:4]
    disc = _disc(sc)
    dev = torch.device("cuda")
    out = disc.linearize_batch_device(*(torch.as_tensor(a, device=dev) for a in (xt0, U, S)))
    torch.cuda.synchronize()
    dev_out = [t.cpu().numpy() for t in out[:4]]
    host_out = disc.linearize_batch(xt0, U, S)
    for a, h, r in zip(dev_out, host_out, ref):
        assert np.array_equal(a, h)
        d = np.abs(a - r).reshape(B, -1).max(axis=1) / (1.0 + np.abs(r).reshape(B, -1).max(axis=1))
        assert d.max() <= TOL, (int(d.argmax()), float(d.max()))
    for a, r in zip(dev_out[1:3], ref[1:3]):  # jx, ju: structural zeros stay exact
        assert np.array_equal(a == 0.0, r == 0.0)
