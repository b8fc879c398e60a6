"""Golden fixtures for implicit terrains with a variable exponent (build container only).

The reference's surface grammar (cito/multibody.py:124-141) admits any sympy.Pow,
including symbolic exponents; the GPU byte-code lowers a**b with a symbolic b to
exp(b log a).  This pins that against the UNMODIFIED reference (jax shim):

  surface_pow.npz   the reference's sinusoid test model (tests/conftest.py:92-101)
                    on the terrain  pz - 0.1*sin(px) - 0.05*(px**2 + 1)**(0.5*cos(px)):
                    Discretizer(model, substeps=5).linearize_batch of 4 seeded intervals

Usage:  python tests/golden/make_golden_surface.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref_runner  # noqa: E402

EXPR = "pz - 0.1*sin(px) - 0.05*(px**2 + 1)**(0.5*cos(px))"


def main():
    ref_runner.import_cito()
    from cito.augmentation import Discretizer
    from cito.multibody import ContactSpec, ImplicitSurface, LinkSpec, RobotModel

    model = RobotModel(links=(LinkSpec(mass=1.0, inertia=0.1),), joints=(),
                       contacts=(ContactSpec(link=0, local_offset=(0.0, 0.0), friction_mu=1.0),),
                       surface=ImplicitSurface(expression=EXPR), gravity=9.81)
    rng = np.random.default_rng(17)
    B = 4
    q = np.stack([rng.uniform(-1, 1, B), rng.uniform(0.05, 0.4, B), rng.normal(0, 0.3, B)], axis=1)
    v = rng.normal(0, 0.5, (B, 3))
    y = rng.uniform(0, 0.1, (B, 5))
    xt0 = np.concatenate([q, v, y], axis=1)
    U = np.concatenate([rng.uniform(-2, 2, (B, 1)), rng.uniform(0, 9.81, (B, 1)), rng.uniform(0, 1, (B, 1))] * 2,
                       axis=1)
    S = rng.uniform(0.02, 0.08, B)
    d = Discretizer(model, substeps=5)
    e, jx, ju, js = d.linearize_batch(xt0, U, S)
    np.savez_compressed(os.path.join(HERE, "surface_pow.npz"), expr=np.array(EXPR), lin_xt0=xt0, lin_U=U, lin_S=S,
                        lin_ends=e, lin_jx=jx, lin_ju=ju, lin_js=js)
    print("done", np.abs(jx).max())


if __name__ == "__main__":
    main()
