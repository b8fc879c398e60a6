"""Robot-model description for the C ABI (``cito_model_desc`` in include/cito_b200.h).

Mirrors the reference's model types (``cito.multibody.RobotModel`` /
``LinkSpec`` / ``JointSpec`` / ``ContactSpec`` / ``FlatSurface`` /
``ImplicitSurface``, /root/reference/pkg/src/cito/multibody.py:53-256) and its
JSON format (``model_from_dict``, multibody.py:432-462), so the GPU path can be
driven either by the reference's own objects (duck-typed) or standalone from
JSON on a box without the reference installed.
"""

import ctypes
import json
from dataclasses import dataclass, field

import numpy as np

MAX_LINKS = 16
MAX_JOINTS = 16
MAX_CONTACTS = 8
MAX_PATH = 48
MAX_GOUT = 48
MAX_EXPR = 256

SURFACE_FLAT = 0
SURFACE_IMPLICIT = 1

OP_CONST, OP_PX, OP_PZ, OP_ADD, OP_MUL, OP_POW, OP_SIN, OP_COS, OP_NEG, OP_LOG, OP_EXP = range(11)

_d2 = ctypes.c_double * 2


class ModelDesc(ctypes.Structure):
    """ctypes mirror of ``cito_model_desc`` (field order must match the header)."""

    _fields_ = [
        ("n_links", ctypes.c_int32),
        ("n_joints", ctypes.c_int32),
        ("n_contacts", ctypes.c_int32),
        ("surface_kind", ctypes.c_int32),
        ("gravity", ctypes.c_double),
        ("surface_height", ctypes.c_double),
        ("link_mass", ctypes.c_double * MAX_LINKS),
        ("link_inertia", ctypes.c_double * MAX_LINKS),
        ("link_com", _d2 * MAX_LINKS),
        ("joint_parent", ctypes.c_int32 * MAX_JOINTS),
        ("joint_child", ctypes.c_int32 * MAX_JOINTS),
        ("joint_actuated", ctypes.c_int32 * MAX_JOINTS),
        ("joint_spring", ctypes.c_int32 * MAX_JOINTS),
        ("joint_parent_anchor", _d2 * MAX_JOINTS),
        ("joint_child_anchor", _d2 * MAX_JOINTS),
        ("joint_stiffness", ctypes.c_double * MAX_JOINTS),
        ("joint_damping", ctypes.c_double * MAX_JOINTS),
        ("joint_rest", ctypes.c_double * MAX_JOINTS),
        ("contact_link", ctypes.c_int32 * MAX_CONTACTS),
        ("contact_offset", _d2 * MAX_CONTACTS),
        ("contact_mu", ctypes.c_double * MAX_CONTACTS),
        ("contact_restitution", ctypes.c_double * MAX_CONTACTS),
        ("n_joint_limits", ctypes.c_int32),
        ("jl_joint", ctypes.c_int32 * MAX_PATH),
        ("jl_lo", ctypes.c_double * MAX_PATH),
        ("jl_hi", ctypes.c_double * MAX_PATH),
        ("n_height_bounds", ctypes.c_int32),
        ("hb_link", ctypes.c_int32 * MAX_PATH),
        ("hb_lo", ctypes.c_double * MAX_PATH),
        ("hb_hi", ctypes.c_double * MAX_PATH),
        ("n_g_out", ctypes.c_int32),
        ("expr_len", ctypes.c_int32),
        ("mixing", ctypes.c_double * (MAX_GOUT * MAX_PATH)),
        ("expr_op", ctypes.c_int32 * MAX_EXPR),
        ("expr_arg", ctypes.c_double * MAX_EXPR),
    ]


class Dims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("n_q", "n_x", "n_u", "n_y", "n_xt", "n_j", "n_a", "n_g", "D")]


# ---------------------------------------------------------------------------
# standalone model types (same fields as the reference's dataclasses)


@dataclass(frozen=True)
class LinkSpec:
    mass: float
    inertia: float
    com_offset: tuple = (0.0, 0.0)
    geometry_length: float = 0.0


@dataclass(frozen=True)
class JointSpec:
    parent_link: int
    child_link: int
    parent_anchor: tuple
    child_anchor: tuple
    stiffness: float = 0.0
    damping: float = 0.0
    rest_angle: float = 0.0
    torque_min: float = 0.0
    torque_max: float = 0.0
    actuated: bool = False


@dataclass(frozen=True)
class ContactSpec:
    link: int
    local_offset: tuple
    friction_mu: float = 1.0
    restitution: float = 0.0


@dataclass(frozen=True)
class FlatSurface:
    height: float = 0.0
    kind: str = field(default="flat", init=False)


@dataclass(frozen=True)
class ImplicitSurface:
    expression: str
    kind: str = field(default="implicit", init=False)


@dataclass(frozen=True, eq=False)
class RobotModel:
    links: tuple
    joints: tuple
    contacts: tuple
    surface: object
    gravity: float = 9.81

    @property
    def n_links(self):
        return len(self.links)

    @property
    def n_q(self):
        return 3 * len(self.links)

    @property
    def n_j(self):
        return 2 * len(self.joints)

    @property
    def n_c(self):
        return len(self.contacts)

    @property
    def n_a(self):
        return sum(1 for j in self.joints if j.actuated)

    @property
    def actuated_joints(self):
        return tuple(i for i, j in enumerate(self.joints) if j.actuated)


def model_from_dict(data):
    """Same schema as cito.multibody.model_from_dict (multibody.py:432-462)."""
    links = tuple(LinkSpec(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})
                  for d in data.get("links", []))
    joints = tuple(JointSpec(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})
                   for d in data.get("joints", []))
    contacts = tuple(ContactSpec(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})
                     for d in data.get("contacts", []))
    sdata = dict(data["surface"])
    kind = sdata.pop("kind")
    if kind == "flat":
        surface = FlatSurface(**sdata)
    elif kind == "implicit":
        surface = ImplicitSurface(**sdata)
    else:
        raise ValueError(f"unknown surface kind: {kind}")
    return RobotModel(links=links, joints=joints, contacts=contacts, surface=surface,
                      gravity=float(data.get("gravity", 9.81)))


def load_model(path):
    with open(path) as f:
        return model_from_dict(json.load(f))


# ---------------------------------------------------------------------------
# implicit-surface expression -> postfix byte-code


def compile_surface_expression(expression):
    """Compile h(px, pz) (reference grammar, multibody.py:124-141) to postfix ops."""
    import sympy

    px, pz = sympy.symbols("px pz")
    expr = sympy.sympify(expression, locals={"sin": sympy.sin, "cos": sympy.cos, "px": px, "pz": pz})
    ops, args = [], []

    def emit(op, arg=0.0):
        ops.append(op)
        args.append(float(arg))

    def walk(e):
        if e == px:
            emit(OP_PX)
        elif e == pz:
            emit(OP_PZ)
        elif e.is_Number:
            emit(OP_CONST, float(e))
        elif isinstance(e, sympy.Add):
            terms = e.args
            walk(terms[0])
            for t in terms[1:]:
                walk(t)
                emit(OP_ADD)
        elif isinstance(e, sympy.Mul):
            fs = e.args
            walk(fs[0])
            for t in fs[1:]:
                walk(t)
                emit(OP_MUL)
        elif isinstance(e, sympy.Pow):
            base, ex = e.args
            if ex.is_Number:
                walk(base)
                emit(OP_POW, float(ex))
            else:  # base**ex = exp(ex * log(base)) (jnp.power for a symbolic exponent)
                walk(ex)
                walk(base)
                emit(OP_LOG)
                emit(OP_MUL)
                emit(OP_EXP)
        elif isinstance(e, sympy.sin):
            walk(e.args[0])
            emit(OP_SIN)
        elif isinstance(e, sympy.cos):
            walk(e.args[0])
            emit(OP_COS)
        else:
            raise ValueError(f"surface expression uses unsupported operation: {e!r}")

    walk(expr)
    if len(ops) > MAX_EXPR:
        raise ValueError("surface expression too long")
    return ops, args


def path_spec_from_fn(path_fn):
    """Recover (joint_angle_limits, body_height_bounds) from the closure built by
    cito.augmentation.build_path_constraints (augmentation.py:100-131)."""
    if path_fn is None:
        return (), ()
    spec = getattr(path_fn, "cito_path_spec", None)
    if spec is not None:
        return tuple(spec[0]), tuple(spec[1])
    code = getattr(path_fn, "__code__", None)
    cells = getattr(path_fn, "__closure__", None) or ()
    names = code.co_freevars if code is not None else ()
    env = {n: c.cell_contents for n, c in zip(names, cells)}
    if "joint_angle_limits" not in env or "body_height_bounds" not in env:
        raise NotImplementedError(
            "path_fn is not a cito.augmentation.build_path_constraints closure; the GPU "
            "path needs the structured path-constraint spec (joint_angle_limits, body_height_bounds)")
    return tuple(env["joint_angle_limits"]), tuple(env["body_height_bounds"])


def build_path_constraints(model, joint_angle_limits=(), body_height_bounds=()):
    """Host marker mirroring cito.augmentation.build_path_constraints: returns
    (g, n_g) where g carries the structured spec for the GPU path (the values
    are computed on the device, so g itself is not evaluated on the host)."""
    joint_angle_limits = tuple(tuple(r) for r in joint_angle_limits)
    body_height_bounds = tuple(tuple(r) for r in body_height_bounds)
    n_g = len(model.contacts) + 2 * len(joint_angle_limits) + 2 * len(body_height_bounds)

    def g(x, u):  # pragma: no cover - marker only
        raise NotImplementedError("path constraints are evaluated on the GPU")

    g.cito_path_spec = (joint_angle_limits, body_height_bounds)
    return g, n_g


def pack_model(model, mixing=None, path_fn=None):
    """Fill a ModelDesc from a RobotModel-like object (reference or standalone)."""
    d = ModelDesc()
    nl, nj, nc = len(model.links), len(model.joints), len(model.contacts)
    if nl < 1 or nl > MAX_LINKS or nj > MAX_JOINTS or nc > MAX_CONTACTS:
        raise ValueError(f"model size outside the compiled limits (links {nl}, joints {nj}, contacts {nc})")
    d.n_links, d.n_joints, d.n_contacts = nl, nj, nc
    d.gravity = float(model.gravity)
    for i, l in enumerate(model.links):
        d.link_mass[i] = float(l.mass)
        d.link_inertia[i] = float(l.inertia)
        d.link_com[i][0], d.link_com[i][1] = (float(c) for c in l.com_offset)
    for i, j in enumerate(model.joints):
        d.joint_parent[i] = int(j.parent_link)
        d.joint_child[i] = int(j.child_link)
        d.joint_actuated[i] = 1 if j.actuated else 0
        d.joint_spring[i] = 1 if (j.stiffness != 0.0 or j.damping != 0.0) else 0
        d.joint_parent_anchor[i][0], d.joint_parent_anchor[i][1] = (float(c) for c in j.parent_anchor)
        d.joint_child_anchor[i][0], d.joint_child_anchor[i][1] = (float(c) for c in j.child_anchor)
        d.joint_stiffness[i] = float(j.stiffness)
        d.joint_damping[i] = float(j.damping)
        d.joint_rest[i] = float(j.rest_angle)
    for i, c in enumerate(model.contacts):
        d.contact_link[i] = int(c.link)
        d.contact_offset[i][0], d.contact_offset[i][1] = (float(v) for v in c.local_offset)
        d.contact_mu[i] = float(c.friction_mu)
        d.contact_restitution[i] = float(c.restitution)
    surf = model.surface
    if getattr(surf, "kind", "flat") == "flat":
        d.surface_kind = SURFACE_FLAT
        d.surface_height = float(surf.height)
    else:
        d.surface_kind = SURFACE_IMPLICIT
        ops, args = compile_surface_expression(surf.expression)
        d.expr_len = len(ops)
        for k, (o, a) in enumerate(zip(ops, args)):
            d.expr_op[k] = o
            d.expr_arg[k] = a
    if mixing is not None:
        mix = np.asarray(mixing, dtype=float)
        if path_fn is None:
            raise ValueError("mixing matrix given without a path-constraint function")
        jl, hb = path_spec_from_fn(path_fn)
        n_g = nc + 2 * len(jl) + 2 * len(hb)
        if mix.ndim != 2 or mix.shape[1] != n_g:
            raise ValueError(f"mixing matrix must have {n_g} columns, got shape {mix.shape}")
        if mix.shape[0] > MAX_GOUT or n_g > MAX_PATH:
            raise ValueError("too many path-constraint rows for the compiled limits")
        d.n_g_out = mix.shape[0]
        d.n_joint_limits = len(jl)
        for k, (ji, lo, hi) in enumerate(jl):
            d.jl_joint[k] = int(ji)
            d.jl_lo[k] = float(lo)
            d.jl_hi[k] = float(hi)
        d.n_height_bounds = len(hb)
        for k, (li, lo, hi) in enumerate(hb):
            d.hb_link[k] = int(li)
            d.hb_lo[k] = float(lo)
            d.hb_hi[k] = float(hi)
        for r in range(mix.shape[0]):
            for c in range(n_g):
                d.mixing[r * MAX_PATH + c] = float(mix[r, c])
    return d


def model_dims(model, n_g_out=0):
    n_q = 3 * len(model.links)
    n_a = sum(1 for j in model.joints if j.actuated)
    n_c = len(model.contacts)
    n_u = n_a + 3 * n_c
    n_y = 5 * n_c + n_g_out
    n_xt = 2 * n_q + n_y
    return dict(n_q=n_q, n_x=2 * n_q, n_u=n_u, n_y=n_y, n_xt=n_xt, n_a=n_a, n_c=n_c,
                D=n_xt + 2 * n_u + 1)
