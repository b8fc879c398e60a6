"""The drop-in boundary on CPU: the C-ABI library loads, exports every symbol
include/cito_b200.h declares, and resolves the reference's models to compiled
topologies with the reference's dimensions (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN_CASES, ROOT, golden_scenario


def test_library_exports_header_symbols():
    from paper_2604_09993_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "cito_b200.h")).read()
    names = sorted(set(re.findall(r"\b(cito_[a-z_]+)\s*\(", hdr)))
    assert len(names) >= 12
    L = ctypes.CDLL(_lib.SO_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert b"sm_100a" in _lib.lib().cito_version()


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_create_resolves_bundled_models(name):
    from paper_2604_09993_b200 import Discretizer
    from paper_2604_09993_b200.scenario import Layout

    sc = golden_scenario(name)
    g, n_g = sc.path_constraints()
    disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
    lay = Layout(sc)
    d = disc._h.dims
    assert (d.n_xt, d.n_u, d.n_y, d.n_q) == (lay.n_xt, lay.n_u, lay.n_y, lay.n_q)
    assert d.D == lay.n_xt + 2 * lay.n_u + 1


def test_python_and_c_topology_keys_agree():
    from paper_2604_09993_b200 import _lib, topology
    from paper_2604_09993_b200.model import pack_model

    for name in GOLDEN_CASES:
        sc = golden_scenario(name)
        g, n_g = sc.path_constraints()
        d = pack_model(sc.model, sc.mixing_matrix(n_g), g)
        assert topology.key_from_desc(d) in topology.compiled_keys()
        _lib.Handle(d, sc.substeps)  # C side finds the same key


def test_constructor_errors():
    from paper_2604_09993_b200 import Discretizer
    from test_reference_models import point_mass_model

    m = point_mass_model()
    with pytest.raises(ValueError):
        Discretizer(m, substeps=0)
    with pytest.raises(ValueError):
        Discretizer(m, mixing=np.eye(1), path_fn=None)


def test_path_spec_from_reference_closure():
    """path_fn built like cito.augmentation.build_path_constraints (augmentation.py:100-131)."""
    from paper_2604_09993_b200.model import path_spec_from_fn

    def build_path_constraints(model, joint_angle_limits=(), body_height_bounds=()):
        joint_angle_limits = tuple(joint_angle_limits)
        body_height_bounds = tuple(body_height_bounds)

        def g(x, u):
            return (model, joint_angle_limits, body_height_bounds)

        return g, 0

    g, _ = build_path_constraints("m", ((0, -1.0, 1.0),), ((2, 0.1, 0.9),))
    assert path_spec_from_fn(g) == (((0, -1.0, 1.0),), ((2, 0.1, 0.9),))
    with pytest.raises(NotImplementedError):
        path_spec_from_fn(lambda x, u: x)


def test_surface_bytecode_matches_sympy():
    import sympy

    from paper_2604_09993_b200.model import compile_surface_expression

    expr = "pz - 0.03*sin(7.853981633974483*px) + 0.2*cos(px)**2"
    ops, args = compile_surface_expression(expr)
    px, pz = sympy.symbols("px pz")
    f = sympy.lambdify((px, pz), sympy.sympify(expr), "math")
    for x, z in ((0.3, 0.1), (-1.2, 2.0)):
        st = []
        for o, a in zip(ops, args):
            if o == 0:
                st.append(a)
            elif o == 1:
                st.append(x)
            elif o == 2:
                st.append(z)
            elif o == 3:
                b_, a_ = st.pop(), st.pop()
                st.append(a_ + b_)
            elif o == 4:
                b_, a_ = st.pop(), st.pop()
                st.append(a_ * b_)
            elif o == 5:
                st.append(st.pop() ** a)
            elif o == 6:
                st.append(np.sin(st.pop()))
            elif o == 7:
                st.append(np.cos(st.pop()))
        assert abs(st[0] - f(x, z)) < 1e-14
