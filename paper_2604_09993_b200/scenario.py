"""Scenario, decision-vector layout and variable scaling (host side).

Mirrors, for the parts the linearize/scatter path needs,
  ScenarioSpec     /root/reference/pkg/src/cito/ocp.py:49-128
  Layout           /root/reference/pkg/src/cito/ocp.py:131-203
  _build_scaling   /root/reference/pkg/src/cito/ocp.py:394-417
  scenario_from_dict / load_scenario  ocp.py:578-664
so that bench.py and the GPU tests can pose the reference's bundled scenarios
on a box where the reference package is not installed.  When the reference's
own ``Transcription`` is available, ``from_transcription`` adapts it instead.
"""

import json
import os
from dataclasses import dataclass

import numpy as np

from . import model as _model


@dataclass(eq=False)
class ScenarioSpec:
    model: object
    x_init: np.ndarray
    x_final: np.ndarray
    t_f: float
    N: int = 15
    substeps: int = 10
    fixed_time: bool = True
    s_bounds: tuple = None
    mask_final: np.ndarray = None
    joint_angle_limits: tuple = ()
    body_height_bounds: tuple = ()
    mixing: str = "identity"
    ctcs_epsilon: float = 1e-4
    torque_weight: float = 1.0
    s_reg: float = 0.0
    force_max: float = None
    impulse_max: float = None
    gamma_max: float = 10.0
    guess_force_scale: float = None
    guess_impulse_scale: float = 0.0
    seed: int = 0

    def __post_init__(self):  # ocp.py:75-105 (joint-consistency check omitted: host-only)
        if self.N < 2:
            raise ValueError("need at least two grid nodes")
        self.x_init = np.asarray(self.x_init, dtype=float)
        self.x_final = np.asarray(self.x_final, dtype=float)
        n_x = 2 * self.model.n_q
        if self.mask_final is None:
            self.mask_final = np.ones(n_x, dtype=bool)
        self.mask_final = np.asarray(self.mask_final, dtype=bool)
        s_nom = self.t_f / (self.N - 1)
        if self.s_bounds is None:
            self.s_bounds = (0.2 * s_nom, 5.0 * s_nom)
        if not (0 < self.s_bounds[0] <= s_nom <= self.s_bounds[1]):
            raise ValueError("s_bounds must bracket the nominal dilation")
        weight = sum(l.mass for l in self.model.links) * max(abs(self.model.gravity), 1.0)
        if self.force_max is None:
            self.force_max = 10.0 * weight
        if self.impulse_max is None:
            self.impulse_max = 2.0 * weight * s_nom
        if self.guess_force_scale is None:
            self.guess_force_scale = weight

    @property
    def s_nominal(self):
        return self.t_f / (self.N - 1)

    def mixing_matrix(self, n_g):  # ocp.py:121-126
        if self.mixing == "identity":
            return np.eye(n_g) if n_g else None
        if self.mixing == "ones":
            return np.ones((1, n_g)) if n_g else None
        raise ValueError(f"unknown mixing mode {self.mixing!r}")

    def path_constraints(self):
        return _model.build_path_constraints(self.model, self.joint_angle_limits, self.body_height_bounds)


def scenario_from_dict(data, base_dir="."):  # ocp.py:578-624
    m = data["model"]
    if isinstance(m, str):
        model = _model.load_model(os.path.join(base_dir, m))
    else:
        model = _model.model_from_dict(m)
    horizon = data["horizon"]
    path = data.get("path_constraints", {})
    cost = data.get("cost", {})
    bounds = data.get("bounds", {})
    kw = {}
    if "s_min" in horizon or "s_max" in horizon:
        kw["s_bounds"] = (horizon["s_min"], horizon["s_max"])
    if "mask_final" in data:
        kw["mask_final"] = np.asarray(data["mask_final"], dtype=bool)
    return ScenarioSpec(
        model=model,
        x_init=np.asarray(data["x_init"], dtype=float),
        x_final=np.asarray(data["x_final"], dtype=float),
        t_f=float(horizon["t_f"]),
        fixed_time=bool(horizon.get("fixed", True)),
        N=int(data.get("N", 15)),
        substeps=int(data.get("substeps", 10)),
        joint_angle_limits=tuple(tuple(r) for r in path.get("joint_angle_limits", ())),
        body_height_bounds=tuple(tuple(r) for r in path.get("body_height_bounds", ())),
        mixing=path.get("mixing", "identity"),
        ctcs_epsilon=float(data.get("ctcs_epsilon", 1e-4)),
        torque_weight=float(cost.get("torque_weight", 1.0)),
        s_reg=float(cost.get("s_reg", 0.0)),
        force_max=bounds.get("force_max"),
        impulse_max=bounds.get("impulse_max"),
        gamma_max=float(bounds.get("gamma_max", 10.0)),
        guess_force_scale=bounds.get("guess_force_scale"),
        guess_impulse_scale=float(bounds.get("guess_impulse_scale", 0.0)),
        seed=int(data.get("seed", 0)),
        **kw,
    )


def load_scenario(path, **overrides):
    """Load a scenario file; overrides follow the reference's recipe
    ``dataclasses.replace(sc, N=N, s_bounds=None)``: derived
    fields already filled by __post_init__ (force_max, impulse_max,
    guess_force_scale) keep the values of the file's own N."""
    from dataclasses import replace

    with open(path) as f:
        data = json.load(f)
    sc = scenario_from_dict(data, base_dir=os.path.dirname(os.path.abspath(path)))
    if "N" in overrides:
        sc = replace(sc, N=int(overrides.pop("N")), s_bounds=None)
    if "substeps" in overrides:
        sc = replace(sc, substeps=int(overrides.pop("substeps")))
    if overrides:
        raise TypeError(f"unknown overrides {sorted(overrides)}")
    return sc


class Layout:
    """Decision-vector index map, identical order to cito.ocp.Layout (ocp.py:131-203)."""

    def __init__(self, scenario):
        model = scenario.model
        self.N = N = scenario.N
        self.n_q = model.n_q
        g, n_g = scenario.path_constraints()
        mix = scenario.mixing_matrix(n_g)
        self.n_g_out = 0 if mix is None else mix.shape[0]
        self.n_y = 5 * model.n_c + self.n_g_out
        self.n_xt = 2 * model.n_q + self.n_y
        self.n_u = model.n_a + 3 * model.n_c
        self.n_c = model.n_c
        self.n_a = model.n_a
        nxt, nu, nc = self.n_xt, self.n_u, self.n_c
        self.xm_off = np.array([2 * k * nxt for k in range(N)], dtype=np.int64)
        self.xp_off = self.xm_off + nxt
        base_u = 2 * N * nxt
        self.u_off = np.array([base_u + k * (2 * nu + 1) for k in range(N - 1)], dtype=np.int64)
        self.s_off = self.u_off + 2 * nu
        base_p = base_u + (N - 1) * (2 * nu + 1)
        self.phi_off = np.array([base_p + k * 3 * nc for k in range(N)], dtype=np.int64)
        self.gam_off = self.phi_off + 2 * nc
        self.dim = base_p + N * 3 * nc

    def xm(self, k):
        return np.arange(self.xm_off[k], self.xm_off[k] + self.n_xt)

    def xp(self, k):
        return np.arange(self.xp_off[k], self.xp_off[k] + self.n_xt)

    def u(self, k):
        return np.arange(self.u_off[k], self.u_off[k] + 2 * self.n_u)

    def s(self, k):
        return np.arange(self.s_off[k], self.s_off[k] + 1)

    def phi(self, k):
        return np.arange(self.phi_off[k], self.phi_off[k] + 2 * self.n_c)

    def gam(self, k):
        return np.arange(self.gam_off[k], self.gam_off[k] + self.n_c)

    def y_of_xm(self, k):
        return self.xm(k)[2 * self.n_q:]

    def y_of_xp(self, k):
        return self.xp(k)[2 * self.n_q:]


def build_scaling(scenario, lay):
    """sigma of z_phys = sigma * z_scaled (ocp.py:394-417); returns (scale_v, state_scale, u_scale)."""
    model = scenario.model
    n_q = lay.n_q
    scale_v = np.ones(lay.dim)
    state_scale = np.ones(lay.n_xt)
    for i in range(2 * n_q):
        state_scale[i] = max(1.0, abs(scenario.x_init[i]), abs(scenario.x_final[i]))
    u_scale = np.ones(lay.n_u)
    tq = [max(abs(model.joints[j].torque_min), abs(model.joints[j].torque_max), 1e-9)
          for j in model.actuated_joints]
    u_scale[: lay.n_a] = tq
    u_scale[lay.n_a: lay.n_a + 2 * lay.n_c] = scenario.force_max
    u_scale[lay.n_a + 2 * lay.n_c:] = scenario.gamma_max
    for k in range(lay.N):
        scale_v[lay.xm(k)] = state_scale
        scale_v[lay.xp(k)] = state_scale
        scale_v[lay.phi(k)] = scenario.impulse_max
        scale_v[lay.gam(k)] = scenario.gamma_max
    for k in range(lay.N - 1):
        scale_v[lay.u(k)] = np.concatenate([u_scale, u_scale])
        scale_v[lay.s(k)] = scenario.s_nominal
    return scale_v, state_scale, u_scale


def assets_dir():
    """Model/scenario JSON assets (data copied from the reference by tests/golden/make_golden.py)."""
    here = os.path.dirname(os.path.abspath(__file__))
    return os.path.join(os.path.dirname(here), "tests", "golden", "assets")


def bundled(name, **overrides):
    return load_scenario(os.path.join(assets_dir(), f"{name}.json"), **overrides)
