"""The reference's own hot-path tests, re-expressed against the GPU Discretizer.

Models are the fixtures of /root/reference/pkg/tests/conftest.py:14-101
(rebuilt with the standalone model types, same numbers).  Each test cites the
reference test it restates.
"""

import numpy as np
import pytest

from conftest import rel_err

from paper_2604_09993_b200.model import (ContactSpec, FlatSurface, ImplicitSurface, JointSpec, LinkSpec,
                                         RobotModel, build_path_constraints)


def free_link_model(gravity=9.81):
    return RobotModel(links=(LinkSpec(mass=2.0, inertia=0.5, geometry_length=1.0),), joints=(), contacts=(),
                      surface=FlatSurface(height=-100.0), gravity=gravity)


def point_mass_model(gravity=9.81):
    return RobotModel(links=(LinkSpec(mass=1.0, inertia=0.1),), joints=(),
                      contacts=(ContactSpec(link=0, local_offset=(0.0, 0.0), friction_mu=1.0),),
                      surface=FlatSurface(height=0.0), gravity=gravity)


def pendulum_model():
    return RobotModel(links=(LinkSpec(mass=2.0, inertia=2.0 / 12.0, geometry_length=1.0),),
                      joints=(JointSpec(parent_link=-1, child_link=0, parent_anchor=(0.0, 0.0),
                                        child_anchor=(-0.5, 0.0), actuated=False),),
                      contacts=(), surface=FlatSurface(height=-100.0), gravity=9.81)


def double_pendulum_model():
    link = LinkSpec(mass=1.0, inertia=1.0 / 12.0, geometry_length=1.0)
    return RobotModel(links=(link, link),
                      joints=(JointSpec(parent_link=-1, child_link=0, parent_anchor=(0.0, 0.0),
                                        child_anchor=(-0.5, 0.0)),
                              JointSpec(parent_link=0, child_link=1, parent_anchor=(0.5, 0.0),
                                        child_anchor=(-0.5, 0.0), actuated=True, torque_min=-10.0,
                                        torque_max=10.0)),
                      contacts=(), surface=FlatSurface(height=-100.0), gravity=9.81)


def sinusoid_model():
    return RobotModel(links=(LinkSpec(mass=1.0, inertia=0.1),), joints=(),
                      contacts=(ContactSpec(link=0, local_offset=(0.0, 0.0), friction_mu=1.0),),
                      surface=ImplicitSurface(expression="pz - 0.1*sin(px)"), gravity=9.81)


def spring_pendulum_model():
    """double pendulum with a spring/damper on the actuated joint (multibody.py:315-317)."""
    link = LinkSpec(mass=1.0, inertia=1.0 / 12.0, com_offset=(0.05, -0.02), geometry_length=1.0)
    return RobotModel(links=(link, link),
                      joints=(JointSpec(parent_link=-1, child_link=0, parent_anchor=(0.1, 0.0),
                                        child_anchor=(-0.5, 0.0)),
                              JointSpec(parent_link=0, child_link=1, parent_anchor=(0.5, 0.0),
                                        child_anchor=(-0.5, 0.0), actuated=True, torque_min=-10.0,
                                        torque_max=10.0, stiffness=3.0, damping=0.4, rest_angle=0.2)),
                      contacts=(), surface=FlatSurface(height=-100.0), gravity=9.81)


# --------------------------------------------------------------------------- CPU: oracle vs closed forms
def test_oracle_constant_flow_exact():
    """tests/test_augmentation.py:84-102 on the C oracle (the checker itself)."""
    import pyoracle
    from paper_2604_09993_b200.model import pack_model

    d = pack_model(free_link_model(gravity=0.0))
    e, jx, ju, js, _ = pyoracle.linearize(d, 10, np.zeros((1, 6)), np.zeros((1, 0)), [1.0])
    exp = np.eye(6)
    exp[:3, 3:] = np.eye(3)
    assert np.allclose(e[0], 0.0, atol=1e-14) and np.allclose(jx[0], exp, atol=1e-12)


# --------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_constant_flow_exact():
    """tests/test_augmentation.py:84-102."""
    from paper_2604_09993_b200 import AugmentedState, Discretizer, IntervalParameterization

    disc = Discretizer(free_link_model(gravity=0.0))
    start = AugmentedState(q=np.zeros(3), v=np.zeros(3), y=np.zeros(0))
    res = disc.integrate(start, IntervalParameterization(U=np.zeros((2, 0)), S=1.0))
    assert np.allclose(res.end_state.flat(), start.flat(), atol=1e-14)
    expected = np.eye(6)
    expected[:3, 3:] = np.eye(3)
    assert np.allclose(res.jac_state, expected, atol=1e-12)
    res0 = disc.integrate(start, IntervalParameterization(U=np.zeros((2, 0)), S=0.0))
    assert np.allclose(res0.jac_state, np.eye(6), atol=1e-12)


@pytest.mark.gpu
def test_constant_integrand_exact():
    """tests/test_augmentation.py:104-110."""
    from paper_2604_09993_b200 import AugmentedState, Discretizer, IntervalParameterization

    disc = Discretizer(point_mass_model(gravity=0.0))
    start = AugmentedState(q=np.zeros(3), v=np.zeros(3), y=np.zeros(5))
    U = np.array([[0.0, 1.0, 0.0], [0.0, 1.0, 0.0]])
    res = disc.integrate(start, IntervalParameterization(U=U, S=0.5))
    assert res.end_state.y[0] == pytest.approx(0.5, abs=1e-12)
    assert res.end_state.y[1] == pytest.approx(0.0, abs=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("mk,substeps", [(point_mass_model, 5), (sinusoid_model, 4), (double_pendulum_model, 6),
                                         (spring_pendulum_model, 3), (pendulum_model, 7)])
def test_jacobians_match_fd(mk, substeps):
    """tests/test_augmentation.py:112-141 (rtol 1e-6, atol 1e-7) on more models."""
    from paper_2604_09993_b200 import Discretizer

    m = mk()
    if m.contacts:
        g, n_g = build_path_constraints(m)
        disc = Discretizer(m, np.eye(n_g), g, substeps=substeps)
    else:
        disc = Discretizer(m, substeps=substeps)
    rng = np.random.default_rng(20)
    n_q = m.n_q
    xt0 = np.concatenate([np.array([0.0, 1.0, 0.1] * m.n_links) + rng.normal(size=n_q) * 0.1,
                          rng.normal(size=n_q) * 0.1, np.zeros(disc.n_y)])
    U = rng.uniform(0, 1, size=(2, disc.n_u))
    S = 0.3
    e, jx, ju, js = disc.linearize_batch(xt0[None], U.reshape(1, -1), [S])
    h = 1e-6
    for i in range(len(xt0)):
        xp, xm = xt0.copy(), xt0.copy()
        xp[i] += h
        xm[i] -= h
        fd = (disc.propagate(xp, U, S) - disc.propagate(xm, U, S)) / (2 * h)
        assert np.allclose(jx[0][:, i], fd, rtol=1e-6, atol=1e-7), i
    Uf = U.reshape(-1)
    for i in range(Uf.size):
        up, um = Uf.copy(), Uf.copy()
        up[i] += h
        um[i] -= h
        fd = (disc.propagate(xt0, up, S) - disc.propagate(xt0, um, S)) / (2 * h)
        assert np.allclose(ju[0][:, i], fd, rtol=1e-6, atol=1e-7), i
    fd = (disc.propagate(xt0, U, S + h) - disc.propagate(xt0, U, S - h)) / (2 * h)
    assert np.allclose(js[0], fd, rtol=1e-6, atol=1e-7)


@pytest.mark.gpu
@pytest.mark.parametrize("mk", [double_pendulum_model, spring_pendulum_model, sinusoid_model, pendulum_model])
def test_small_models_vs_oracle(mk):
    """Every compiled test topology against the C oracle at rel 1e-9."""
    import pyoracle
    from paper_2604_09993_b200 import Discretizer
    from paper_2604_09993_b200.model import pack_model

    m = mk()
    if m.contacts:
        g, n_g = build_path_constraints(m)
        mix = np.eye(n_g)
    else:
        g, mix = None, None
    disc = Discretizer(m, mix, g, substeps=5)
    rng = np.random.default_rng(7)
    B = 40
    xt0 = np.concatenate([rng.normal(size=(B, m.n_q)) * 0.5 + np.array([0.0, 1.0, 0.0] * m.n_links),
                          rng.normal(size=(B, m.n_q)) * 0.5, rng.uniform(0, 0.1, size=(B, disc.n_y))], axis=1)
    U = rng.normal(size=(B, 2 * disc.n_u))
    S = rng.uniform(0.05, 0.3, size=B)
    ref = pyoracle.linearize(pack_model(m, mix, g), 5, xt0, U, S)
    out = disc.linearize_batch(xt0, U, S)
    for a, r in zip(out, ref[:4]):
        assert rel_err(a, r) <= 1e-9


@pytest.mark.gpu
def test_y_nondecreasing():
    """tests/test_augmentation.py:143-156."""
    from paper_2604_09993_b200 import Discretizer

    m = point_mass_model()
    g, n_g = build_path_constraints(m)
    disc = Discretizer(m, np.eye(n_g), g)
    rng = np.random.default_rng(21)
    for _ in range(10):
        xt0 = np.concatenate([[0.0, rng.uniform(0.5, 2.0), 0.0], np.zeros(3), np.zeros(6)])
        phi_n = rng.uniform(0, 2)
        phi_t = rng.uniform(-phi_n, phi_n)
        gam = rng.uniform(0, 1)
        U = np.array([[phi_t, phi_n, gam], [phi_t, phi_n, gam]])
        end = disc.propagate(xt0, U, 0.2)
        assert np.all(end[6:11] - xt0[6:11] >= -1e-12)


@pytest.mark.gpu
def test_convergence_order():
    """tests/test_augmentation.py:187-199 (order >= 4)."""
    from paper_2604_09993_b200 import Discretizer

    m = pendulum_model()
    xt0 = np.array([0.5, 0.0, 0.0, 0.0, 0.0, 0.0])
    U = np.zeros((2, 0))
    e5, e10, e20 = (Discretizer(m, substeps=s).propagate(xt0, U, 1.0) for s in (5, 10, 20))
    order = np.log2(np.linalg.norm(e5 - e20) / np.linalg.norm(e10 - e20))
    assert order >= 4.0


@pytest.mark.gpu
def test_ballistic_parabola_exact():
    """tests/test_acceptance.py:527-530."""
    from paper_2604_09993_b200 import Discretizer

    m = RobotModel(links=(LinkSpec(mass=1.0, inertia=0.1),), joints=(), contacts=(),
                   surface=FlatSurface(height=-100.0), gravity=9.81)
    end = Discretizer(m, substeps=5).propagate(np.array([0.0, 0.0, 0.0, 1.0, 2.0, 0.0]), np.zeros((2, 0)), 0.5)
    assert abs(end[1] - (2.0 * 0.5 - 0.5 * 9.81 * 0.25)) <= 1e-10


@pytest.mark.gpu
def test_ind_directional_fd_pointmass_rest():
    """tests/test_acceptance.py:244-264: 50 random points, directional FD, _rel_err <= 1e-5."""
    from conftest import golden_scenario
    from paper_2604_09993_b200 import Discretizer

    sc = golden_scenario("pointmass_rest")
    g, n_g = sc.path_constraints()
    disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
    rng = np.random.default_rng(4)
    h = 1e-6
    n_xt, n_u = disc.n_xt, disc.n_u
    for _ in range(50):
        xt0 = 0.3 * rng.normal(size=n_xt)
        xt0[6:] = np.abs(xt0[6:])
        U = 2.0 * rng.normal(size=(2, n_u))
        S = 0.15 + 0.05 * rng.random()
        dx = rng.normal(size=n_xt)
        dU = rng.normal(size=(2, n_u))
        dS = rng.normal()
        ends, jx, ju, js = disc.linearize_batch(xt0[None], U.reshape(1, -1), [S])
        pred = jx[0] @ dx + ju[0] @ dU.reshape(-1) + js[0] * dS
        fp = disc.propagate(xt0 + h * dx, U + h * dU, S + h * dS)
        fm = disc.propagate(xt0 - h * dx, U - h * dU, S - h * dS)
        assert rel_err((fp - fm) / (2 * h), pred) <= 1e-5


def test_unsupported_topology_fails_loudly(monkeypatch):
    """With the run-time topology build switched off (CITO_JIT=0) a topology outside
    the bundled library raises instead of silently falling back."""
    from paper_2604_09993_b200 import Discretizer
    from paper_2604_09993_b200._lib import UnsupportedModelError

    monkeypatch.setenv("CITO_JIT", "0")

    link = LinkSpec(mass=1.0, inertia=0.1)
    m = RobotModel(links=(link, link, link), joints=(JointSpec(-1, 0, (0, 0), (0, 0)), JointSpec(0, 1, (0, 0), (0, 0)),
                                                     JointSpec(1, 2, (0, 0), (0, 0))),
                   contacts=(), surface=FlatSurface(), gravity=9.81)
    with pytest.raises(UnsupportedModelError):
        Discretizer(m)


# --------------------------------------------------------------------------- rate-level reference tests
def _rate(disc, xt, u):
    """The augmented rate [q'; v'; Omega](x, u) from the GPU path itself: at S = 0 every
    stage input equals the start state, so d(end)/dS = sum_substeps h sum_i b_i f = f
    (augmentation.py:195-211 with constant control)."""
    n_u = disc.n_u
    U = np.concatenate([u, u]).reshape(1, 2 * n_u)
    _, _, _, js = disc.linearize_batch(np.asarray(xt)[None], U, [0.0])
    return js[0]


@pytest.mark.gpu
def test_dilation_consistency():
    """tests/test_augmentation.py:158-185: integrating with dilation S equals integrating
    the undilated system over [0, S] with the same number of steps (manual RKF
    comparator with the same stage recursion, FOH control evaluated at t / S)."""
    from paper_2604_09993_b200 import Discretizer

    m = point_mass_model()
    g, n_g = build_path_constraints(m)
    disc = Discretizer(m, np.eye(n_g), g, substeps=8)
    xt0 = np.concatenate([[0.0, 1.0, 0.2], [0.3, 0.0, 0.0], np.zeros(6)])
    U = np.array([[0.1, 0.5, 0.1], [0.2, 0.3, 0.0]])
    S = 0.7
    end_dilated = disc.propagate(xt0, U, S)
    A = [[], [1 / 4], [3 / 32, 9 / 32], [1932 / 2197, -7200 / 2197, 7296 / 2197],
         [439 / 216, -8.0, 3680 / 513, -845 / 4104], [-8 / 27, 2.0, -3544 / 2565, 1859 / 4104, -11 / 40]]
    Bw = [16 / 135, 0.0, 6656 / 12825, 28561 / 56430, -9 / 50, 2 / 55]
    C = [0.0, 1 / 4, 3 / 8, 12 / 13, 1.0, 1 / 2]  # the RKF tableau (cito/augmentation.py:46-56)
    h = S / 8
    xt = xt0.copy()
    for step in range(8):
        ks = []
        for stage in range(6):
            xs = xt.copy()
            for j, a in enumerate(A[stage]):
                xs = xs + h * a * ks[j]
            tau = (step * h + C[stage] * h) / S
            ks.append(_rate(disc, xs, (1.0 - tau) * U[0] + tau * U[1]))
        xt = xt + h * sum(b * k for b, k in zip(Bw, ks))
    assert np.allclose(end_dilated, xt, atol=1e-9)


@pytest.mark.gpu
def test_pendulum_closed_form():
    """tests/test_acceptance.py:490-503: theta'' = -1.5 g / L cos(theta) at 20 random
    consistent states of the pinned pendulum (rate from the GPU kernel)."""
    from paper_2604_09993_b200 import Discretizer

    m = pendulum_model()
    disc = Discretizer(m, substeps=5)
    rng = np.random.default_rng(8)
    L = 1.0
    for _ in range(20):
        th = rng.uniform(-np.pi, np.pi)
        w = rng.normal()
        q = np.array([0.5 * L * np.cos(th), 0.5 * L * np.sin(th), th])
        v = np.array([-0.5 * L * np.sin(th) * w, 0.5 * L * np.cos(th) * w, w])
        f = _rate(disc, np.concatenate([q, v]), np.zeros(0))
        assert abs(f[5] - (-1.5 * m.gravity / L * np.cos(th))) <= 1e-9


@pytest.mark.gpu
def test_aux_rate_channels():
    """tests/test_augmentation.py:30-58: Omega channel values.  Inactive contact at
    height 0.3: Omega = [0, 0, 0, 0, srelu(0.3)], path channel srelu(-0.3); unit
    normal force -> channel 0 = 1; a structured path row with value 0.5 (a link
    height bound lo - p_z = 0.5; the reference's lambda g(x, u) = [0.5] has no
    device form) passes srelu(0.5) = 0.30902 straight through identity mixing."""
    from paper_2604_09993_b200 import Discretizer

    srelu = lambda x: 0.5 * (x + np.sqrt(x * x + 1.0) - 1.0)  # noqa: E731  (smoothmath.py:60-63)
    m = point_mass_model()
    g, n_g = build_path_constraints(m)
    disc = Discretizer(m, np.eye(n_g), g, substeps=5)
    f = _rate(disc, np.concatenate([[0.0, 0.3, 0.0, 0.0, 0.0, 0.0], np.zeros(6)]), np.zeros(3))
    yd = f[6:]
    assert np.allclose(yd[:4], 0.0, atol=1e-14)
    assert yd[4] == pytest.approx(srelu(0.3), abs=1e-14)
    assert yd[5] == pytest.approx(srelu(-0.3), abs=1e-14)
    f = _rate(disc, np.zeros(12), np.array([0.0, 1.0, 0.0]))
    assert f[6] == pytest.approx(1.0)
    g2, n_g2 = build_path_constraints(m, body_height_bounds=((0, 0.5, 10.0),))
    disc2 = Discretizer(m, np.eye(n_g2), g2, substeps=5)
    f = _rate(disc2, np.zeros(6 + 5 + n_g2), np.zeros(3))
    assert f[6 + 5 + 1] == pytest.approx(srelu(0.5), abs=1e-12)
    assert f[6 + 5 + 1] == pytest.approx(0.30902, abs=1e-5)


@pytest.mark.gpu
def test_node_constraint_jacobians_directional_fd():
    """tests/test_acceptance.py:266-304: the K3 node Jacobians against central
    differences of the K3 node values, pointmass_rest, 50 random points (seed 5),
    h = 1e-6, delta = 0.05, the reference's _rel_err <= 1e-5."""
    import torch

    from conftest import golden_scenario

    from paper_2604_09993_b200.linearize import GpuTranscription

    sc = golden_scenario("pointmass_rest")
    gt = GpuTranscription(sc)
    lay = gt.lay
    rng = np.random.default_rng(5)
    h, delta = 1e-6, 0.05
    n_q = lay.n_q

    def nodes(z):
        r = gt.linearize_device(torch.as_tensor(z, device=gt.device), delta)
        torch.cuda.synchronize()
        return {k: r[k].cpu().numpy() for k in ("psi", "theta", "imp_v", "psi_jac", "theta_jac", "imp_jac")}

    for _ in range(50):
        z = 0.5 * rng.normal(size=lay.dim)
        d = rng.normal(size=lay.dim)
        J, p, mn = nodes(z), nodes(z + h * d), nodes(z - h * d)
        fd_psi = (p["psi"] - mn["psi"]) / (2 * h)
        for k in range(lay.N - 1):
            dy = np.concatenate([d[lay.y_of_xp(k)], d[lay.y_of_xm(k + 1)]])
            assert rel_err(fd_psi[k], J["psi_jac"][k] @ dy) <= 1e-5
        fd_th = (p["theta"] - mn["theta"]) / (2 * h)
        fd_imp = (p["imp_v"] - mn["imp_v"]) / (2 * h)
        for k in range(lay.N):
            dvec = np.concatenate([d[lay.xm(k)][:n_q], d[lay.xm(k)][n_q: 2 * n_q], d[lay.xp(k)][n_q: 2 * n_q],
                                   d[lay.phi(k)], d[lay.gam(k)]])
            assert rel_err(fd_th[k], J["theta_jac"][k] @ dvec) <= 1e-5
            # imp_v = v+ - impact_map(...): the reference's impulse_defect velocity rows
            assert rel_err(fd_imp[k], J["imp_jac"][k] @ dvec[: J["imp_jac"].shape[2]]) <= 1e-5
