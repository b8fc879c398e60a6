"""Deterministic synthetic interval inputs (SURVEY.md §8(d) "Synthetic inputs").

States   alpha ~ U(0,1); q = lerp(x_init, x_final, alpha)[q] + N(0, 0.05^2);
         v ~ N(0, 0.5^2); y ~ U(0, 0.1)
Controls per endpoint: tau ~ 0.5*U(tau_min, tau_max); phi_n ~ U(0, W) with
         W = guess_force_scale (cito/ocp.py:97-103); phi_t ~ U(-mu phi_n, mu phi_n);
         gamma ~ U(0, 1)
Dilation S = s_nom * U(0.5, 2), inside the default bounds [0.2, 5] s_nom (ocp.py:92-96).
"""

import numpy as np


DIVERGED = 1e6  # |end state| above this = the fixed-step integration blew up


def well_posed(ends):
    """Accept mask for random draws: finite and not diverged.  Random states of the
    joint-constrained models at large dilation can make the explicit RK flow blow
    up to |x| ~ 1e20..1e300 while staying finite; such intervals are chaotic
    (rounding is amplified by ||Phi|| ~ 1e30+) and carry no parity information."""
    ends = np.asarray(ends)
    return np.all(np.isfinite(ends), axis=1) & (np.max(np.abs(np.nan_to_num(ends, nan=np.inf)), axis=1) < DIVERGED)


def random_intervals(scenario, B, seed=0, finite_fn=None, max_rounds=50):
    """Seeded synthetic batch.  ``finite_fn(xt0, U, S) -> bool mask`` (e.g. a GPU
    propagate) triggers re-drawing of intervals whose end state is non-finite
    (SURVEY.md §8(d)); the number of re-drawn intervals is returned as 4th value
    when ``finite_fn`` is given."""
    xt0, U, S = _draw(scenario, B, np.random.default_rng(seed))
    if finite_fn is None:
        return xt0, U, S
    redrawn = 0
    rng = np.random.default_rng(seed + 7919)
    for _ in range(max_rounds):
        ok = np.asarray(finite_fn(xt0, U, S), dtype=bool)
        bad = np.where(~ok)[0]
        if bad.size == 0:
            return xt0, U, S, redrawn
        redrawn += bad.size
        x2, U2, S2 = _draw(scenario, bad.size, rng)
        xt0[bad], U[bad], S[bad] = x2, U2, S2
    raise RuntimeError("could not draw finite synthetic intervals")


def _draw(scenario, B, rng):
    model = scenario.model
    n_q = model.n_q
    n_c = len(model.contacts)
    n_a = model.n_a
    n_u = n_a + 3 * n_c
    n_g = n_c + 2 * len(scenario.joint_angle_limits) + 2 * len(scenario.body_height_bounds)
    mix = scenario.mixing_matrix(n_g)
    n_y = 5 * n_c + (0 if mix is None else mix.shape[0])
    n_xt = 2 * n_q + n_y
    alpha = rng.uniform(0.0, 1.0, size=(B, 1))
    q = (1.0 - alpha) * scenario.x_init[None, :n_q] + alpha * scenario.x_final[None, :n_q]
    q = q + rng.normal(0.0, 0.05, size=(B, n_q))
    v = rng.normal(0.0, 0.5, size=(B, n_q))
    y = rng.uniform(0.0, 0.1, size=(B, n_y))
    xt0 = np.concatenate([q, v, y], axis=1)
    U = np.zeros((B, 2, n_u))
    act = [model.joints[j] for j in model.actuated_joints]
    for side in range(2):
        for a, jt in enumerate(act):
            U[:, side, a] = 0.5 * rng.uniform(jt.torque_min, jt.torque_max, size=B)
        for i, c in enumerate(model.contacts):
            fn = rng.uniform(0.0, scenario.guess_force_scale, size=B)
            ft = rng.uniform(-c.friction_mu * fn, c.friction_mu * fn)
            U[:, side, n_a + 2 * i] = ft
            U[:, side, n_a + 2 * i + 1] = fn
        U[:, side, n_a + 2 * n_c:] = rng.uniform(0.0, 1.0, size=(B, n_c))
    S = scenario.s_nominal * rng.uniform(0.5, 2.0, size=B)
    return xt0, U.reshape(B, 2 * n_u), S
