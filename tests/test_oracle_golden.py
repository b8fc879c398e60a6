"""Pin the C oracle (oracle/cito_oracle.c) against vectors produced by the
UNMODIFIED reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import pyoracle
from conftest import rel_err, scenario_desc

TOL = 1e-11  # reference (torch.func AD under the shim) vs plain-C dual numbers: both fp64


def test_linearize_random_points(golden_case):
    name, g, sc = golden_case
    desc = scenario_desc(sc)
    e, jx, ju, js, bad = pyoracle.linearize(desc, int(g["substeps"]), g["lin_xt0"], g["lin_U"], g["lin_S"])
    assert not bad.any()
    for a, k in ((e, "lin_ends"), (jx, "lin_jx"), (ju, "lin_ju"), (js, "lin_js")):
        assert rel_err(a, g[k]) <= TOL, (name, k, rel_err(a, g[k]))


def test_linearize_initial_guess(golden_case):
    name, g, sc = golden_case
    from paper_2604_09993_b200.scenario import Layout

    lay = Layout(sc)
    z = g["ig_z"]
    starts = np.stack([z[lay.xp(k)] for k in range(lay.N - 1)])
    Us = np.stack([z[lay.u(k)] for k in range(lay.N - 1)])
    Ss = np.array([z[lay.s(k)][0] for k in range(lay.N - 1)])
    e, jx, ju, js, bad = pyoracle.linearize(scenario_desc(sc), sc.substeps, starts, Us, Ss)
    for a, k in ((e, "ig_ends"), (jx, "ig_jx"), (ju, "ig_ju"), (js, "ig_js")):
        assert rel_err(a, g[k]) <= TOL, (name, k, rel_err(a, g[k]))
    # structural zero pattern identical (the CSC drops exact zeros, cito/scp.py:190-191)
    for a, k in ((jx, "ig_jx"), (ju, "ig_ju"), (js, "ig_js")):
        assert np.array_equal(a != 0.0, g[k] != 0.0), (name, k)


@pytest.mark.parametrize("which", ["ig", "nd"])
def test_node_relations(golden_case, which):
    name, g, sc = golden_case
    from paper_2604_09993_b200.linearize import node_inputs
    from paper_2604_09993_b200.scenario import Layout

    lay = Layout(sc)
    z = g[f"{which}_z"]
    delta = float(g[f"{which}_delta"])
    y_pairs, theta_vecs = node_inputs(lay, z)
    psi, psi_j, th, th_j, imp, imp_j = pyoracle.node_linearize(scenario_desc(sc), y_pairs, theta_vecs, delta,
                                                               sc.ctcs_epsilon)
    for a, k in ((psi, "psi"), (psi_j, "psi_jac"), (th, "theta"), (th_j, "theta_jac"), (imp, "imp"),
                 (imp_j, "imp_jac")):
        ref = g[f"{which}_{k}"]
        assert a.shape == ref.shape, (k, a.shape, ref.shape)
        assert rel_err(a, ref) <= TOL, (name, which, k, rel_err(a, ref))


def test_oracle_propagate_matches_linearize_ends():
    from conftest import golden_scenario, load_golden

    g = load_golden("halfcheetah_n30")
    sc = golden_scenario("halfcheetah_n30")
    desc = scenario_desc(sc)
    e1, _ = pyoracle.propagate(desc, sc.substeps, g["lin_xt0"], g["lin_U"], g["lin_S"])
    assert rel_err(e1, g["lin_ends"]) <= TOL
