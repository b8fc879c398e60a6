"""Configurable path constraints and run-time compiled topologies.

* Joint-angle-limit and link-height-bound path rows
  (cito/augmentation.py:100-131) with identity and "ones" mixing
  (cito/ocp.py:121-126) on HalfCheetah, against goldens of the unmodified
  reference (tests/golden/make_golden_paths.py): interval linearization,
  linearize_all and the subproblem CSC.  These topologies are not in the bundled
  library, so the GPU path compiles them on first use
  (paper_2604_09993_b200.build.build_topology).
* A model outside every bundled topology (a triple pendulum) built at run time
  into a fresh cache directory, against the oracle.
"""

import os
from dataclasses import replace

import numpy as np
import pytest

import pyoracle
from conftest import GOLDEN, rel_err, scenario_desc

MIXINGS = ["identity", "ones"]
TOL = 1e-9


def _golden(mixing):
    return dict(np.load(os.path.join(GOLDEN, f"halfcheetah_paths_{mixing}.npz")))


def _scenario(g):
    from paper_2604_09993_b200 import scenario as S

    sc = S.bundled("halfcheetah_bound", N=int(g["N"]))
    # (index, lo, hi) triples; the indices come back from the npz as floats
    return replace(sc, joint_angle_limits=tuple((int(r[0]), r[1], r[2]) for r in g["joint_limits"].tolist()),
                   body_height_bounds=tuple((int(r[0]), r[1], r[2]) for r in g["height_bounds"].tolist()),
                   mixing=str(g["mixing"]))


@pytest.mark.parametrize("mixing", MIXINGS)
def test_oracle_matches_reference_path_rows(mixing):
    g = _golden(mixing)
    sc = _scenario(g)
    desc = scenario_desc(sc)
    assert desc.n_joint_limits == 4 and desc.n_height_bounds == 2
    assert desc.n_g_out == (14 if mixing == "identity" else 1)
    e, jx, ju, js, bad = pyoracle.linearize(desc, sc.substeps, g["lin_xt0"], g["lin_U"], g["lin_S"])
    for a, k in ((e, "ends"), (jx, "jx"), (ju, "ju"), (js, "js")):
        assert rel_err(a, g[f"lin_{k}"]) <= 1e-11, k


@pytest.mark.parametrize("mixing", MIXINGS)
def test_path_topologies_are_not_bundled(mixing):
    from paper_2604_09993_b200.topology import compiled_keys, key_from_desc

    sc = _scenario(_golden(mixing))
    assert key_from_desc(scenario_desc(sc)) not in compiled_keys()


def test_jit_topology_compiles():
    """The run-time build cross-compiles here too (nvcc, no GPU); the library lands
    in the in-tree cache so the GPU tests load it instead of rebuilding."""
    from paper_2604_09993_b200 import build
    from paper_2604_09993_b200.topology import entry_from_desc

    for mixing in MIXINGS:
        entry, key = entry_from_desc(scenario_desc(_scenario(_golden(mixing))))
        so = build.build_topology(entry)
        assert os.path.exists(so) and entry[0].startswith("jit_")


@pytest.mark.gpu
@pytest.mark.parametrize("mixing", MIXINGS)
def test_gpu_path_rows_match_reference(mixing):
    from paper_2604_09993_b200 import Discretizer
    from paper_2604_09993_b200.subproblem import GpuSCPStep

    g = _golden(mixing)
    sc = _scenario(g)
    gg, n_g = sc.path_constraints()
    d = Discretizer(sc.model, mixing=sc.mixing_matrix(n_g), path_fn=gg, substeps=sc.substeps)
    out = d.linearize_batch(g["lin_xt0"], g["lin_U"], g["lin_S"])
    for a, k in zip(out, ("ends", "jx", "ju", "js")):
        assert rel_err(a, g[f"lin_{k}"]) <= TOL, k
    step = GpuSCPStep(sc)
    lin, prog, meta = step.iterate(g["ig_z"], 1.0)
    for k in ("ends", "jx", "ju", "js", "defects", "psi", "psi_jac", "theta", "theta_jac", "imp_jac"):
        gk = "ig_imp" if k == "imp_v" else f"ig_{k}"
        assert rel_err(getattr(lin, k), g[gk]) <= TOL, k
    for M in ("A", "G"):
        mat = getattr(prog, M)
        assert np.array_equal(mat.indptr, g[f"sp0_{M}_indptr"]) and np.array_equal(mat.indices,
                                                                                  g[f"sp0_{M}_indices"]), M
        assert rel_err(mat.data, g[f"sp0_{M}_data"]) <= TOL, M
    assert rel_err(prog.b, g["sp0_b"]) <= TOL and rel_err(prog.h, g["sp0_h"]) <= TOL


def _triple_pendulum():
    from paper_2604_09993_b200.model import FlatSurface, JointSpec, LinkSpec, RobotModel

    link = LinkSpec(mass=1.0, inertia=1.0 / 12.0, geometry_length=1.0)
    return RobotModel(links=(link, link, link),
                      joints=(JointSpec(-1, 0, (0.0, 0.0), (-0.5, 0.0)),
                              JointSpec(0, 1, (0.5, 0.0), (-0.5, 0.0), actuated=True, stiffness=2.0, damping=0.1),
                              JointSpec(1, 2, (0.5, 0.0), (-0.5, 0.0), actuated=True)),
                      contacts=(), surface=FlatSurface(height=-100.0), gravity=9.81)


@pytest.mark.gpu
def test_gpu_runtime_built_topology_matches_oracle(tmp_path, monkeypatch):
    """A topology no library carries: the first Discretizer compiles it into a fresh
    cache directory (CITO_JIT_DIR) and the result matches the oracle."""
    from paper_2604_09993_b200 import Discretizer, _lib
    from paper_2604_09993_b200.model import pack_model
    from paper_2604_09993_b200.topology import compiled_keys, key_from_desc

    monkeypatch.setenv("CITO_JIT_DIR", str(tmp_path))
    m = _triple_pendulum()
    desc = pack_model(m)
    assert key_from_desc(desc) not in compiled_keys()
    d = Discretizer(m, substeps=6)
    assert d._h.L is not _lib.lib() and any(p.name.endswith(".so") for p in tmp_path.iterdir())
    rng = np.random.default_rng(7)
    B = 40
    x = np.concatenate([rng.normal(0, 0.3, (B, 9)), rng.normal(0, 0.5, (B, 9))], axis=1)
    U = rng.normal(0, 1.0, (B, 4))
    S = rng.uniform(0.02, 0.08, B)
    ref = pyoracle.linearize(desc, 6, x, U, S)[:4]
    out = d.linearize_batch(x, U, S)
    for a, r in zip(out, ref):
        worst = max(rel_err(a[b], r[b]) for b in range(B))
        assert worst <= TOL
    assert d.launch_count() >= 1


def _pow_surface_model(expr):
    from paper_2604_09993_b200.model import ContactSpec, ImplicitSurface, LinkSpec, RobotModel

    return RobotModel(links=(LinkSpec(mass=1.0, inertia=0.1),), joints=(),
                      contacts=(ContactSpec(link=0, local_offset=(0.0, 0.0), friction_mu=1.0),),
                      surface=ImplicitSurface(expression=expr), gravity=9.81)


def test_variable_exponent_surface_bytecode_and_oracle():
    """a**b with a symbolic exponent (cito/multibody.py:124-141 admits any sympy.Pow)
    lowers to b a LOG MUL EXP; the oracle evaluating that byte-code matches the
    reference's own linearization (golden: tests/golden/make_golden_surface.py)."""
    from paper_2604_09993_b200.model import OP_EXP, OP_LOG, compile_surface_expression, pack_model

    g = dict(np.load(os.path.join(GOLDEN, "surface_pow.npz")))
    ops, _ = compile_surface_expression(str(g["expr"]))
    assert OP_LOG in ops and OP_EXP in ops
    desc = pack_model(_pow_surface_model(str(g["expr"])))
    e, jx, ju, js, bad = pyoracle.linearize(desc, 5, g["lin_xt0"], g["lin_U"], g["lin_S"])
    for a, k in ((e, "ends"), (jx, "jx"), (ju, "ju"), (js, "js")):
        assert rel_err(a, g[f"lin_{k}"]) <= 1e-11, k


@pytest.mark.gpu
def test_gpu_variable_exponent_surface_matches_reference():
    from paper_2604_09993_b200 import Discretizer

    g = dict(np.load(os.path.join(GOLDEN, "surface_pow.npz")))
    d = Discretizer(_pow_surface_model(str(g["expr"])), substeps=5)
    out = d.linearize_batch(g["lin_xt0"], g["lin_U"], g["lin_S"])
    for a, k in zip(out, ("ends", "jx", "ju", "js")):
        assert rel_err(a, g[f"lin_{k}"]) <= TOL, k
