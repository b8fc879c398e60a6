"""GPU replay audit vs the reference's
`cito.verifier.replay_check` (/root/reference/pkg/src/cito/verifier.py:236-346).

Golden rp{tag}_* arrays were produced by running the UNMODIFIED reference
replay_check through the jax shim (tests/golden/make_golden_replay.py).  The
GPU path re-integrates every interval at 10x substeps, chains the FOH segment
propagations and audits every sample on the device; all report fields must
match within the north-star tolerance (rel 1e-9 of fp64 values that went
through integration).
"""

import numpy as np
import pytest

from conftest import golden_scenario, load_golden, rel_err

CASES = [("pointmass_rest", "ig"), ("pointmass_rest", "nd"), ("monoped_n20", "ig"), ("halfcheetah_n30", "ig")]
FIELDS = ["max_penetration", "max_joint_drift", "pair_residuals", "ctcs_increments", "cone_violation",
          "refinement_drift", "cross_products"]


def test_replay_goldens_present():
    for name, tag in CASES:
        g = load_golden(name)
        for f in FIELDS:
            assert f"rp{tag}_{f}" in g, (name, tag, f)
        assert np.all(g[f"rp{tag}_cross_products"] >= 0.0) and float(g[f"rp{tag}_max_penetration"]) >= 0.0


def test_replay_rejects_bad_z():
    from paper_2604_09993_b200.verifier import ReplayAuditor
    from paper_2604_09993_b200.scenario import Layout

    sc = golden_scenario("pointmass_rest")
    aud = ReplayAuditor.__new__(ReplayAuditor)  # shape check happens before any device work
    aud.lay, aud.model = Layout(sc), sc.model
    with pytest.raises(ValueError):
        aud.check(np.zeros(3))


@pytest.mark.gpu
@pytest.mark.parametrize("name,tag", CASES)
def test_gpu_replay_check_matches_reference(name, tag):
    from paper_2604_09993_b200.verifier import replay_check

    g = load_golden(name)
    sc = golden_scenario(name)
    grid = int(g[f"rp{tag}_grid"])
    rep = replay_check(g[f"{tag}_z"], sc.model, sc, grid=grid)
    for f in FIELDS:
        got, ref = np.asarray(getattr(rep, f), dtype=float), g[f"rp{tag}_{f}"]
        assert got.shape == ref.shape, f
        assert rel_err(got, ref) <= 1e-9, (f, rel_err(got, ref))
    assert rep.ctcs_epsilon == float(g[f"rp{tag}_ctcs_epsilon"])


@pytest.mark.gpu
def test_gpu_replay_launches_and_samples():
    """The audit runs on the device: 1 fine + grid segment + 1 audit launches."""
    from paper_2604_09993_b200.verifier import auditor_for

    g = load_golden("monoped_n20")
    sc = golden_scenario("monoped_n20")
    aud = auditor_for(sc)
    n0 = aud.launch_count()
    taus, (fine_end, samples, sds, cj, om) = aud.device_pass(g["ig_z"], 6)
    assert aud.launch_count() - n0 == 1 + 6 + 1
    lay = aud.lay
    assert samples.shape == (7, lay.N - 1, lay.n_xt) and om.shape == (7 * (lay.N - 1), lay.n_y)
    # first sample is the interval start, the last is close to the fine end (same interval, coarser grid)
    z = g["ig_z"]
    assert np.array_equal(samples[0], np.stack([z[lay.xp(k)] for k in range(lay.N - 1)]))
    assert np.all(np.isfinite(samples)) and np.all(np.isfinite(fine_end))
