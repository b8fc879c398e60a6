"""Golden fixtures for configurable path constraints (build container only).

The bundled scenarios only use the per-contact -sd path rows with identity
mixing.  This file pins the other rows of cito.augmentation.build_path_constraints
(augmentation.py:100-131: relative joint-angle limits, link height bounds) and
the "ones" mixing of ScenarioSpec.mixing_matrix (ocp.py:121-126) on HalfCheetah
-- topologies the bundled library does not carry, so the GPU side compiles them
at run time (paper_2604_09993_b200.build.build_topology).

  halfcheetah_paths_<mixing>.npz  for mixing in (identity, ones):
      lin_*   Discretizer.linearize_batch of 3 seeded synthetic intervals
      ig_*    linearize_all at the scenario's initial guess (N = 8)
      sp0_*   build_subproblem -> canonicalize there (delta = 1)
all computed by the UNMODIFIED reference through the jax shim (oracle/ref_runner.py).

Usage:  python tests/golden/make_golden_paths.py
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import ref_runner  # noqa: E402

from paper_2604_09993_b200 import synth  # noqa: E402

# (joint_index, lo, hi) and (link_index, lo, hi) triples (augmentation.py:104-106)
JOINT_LIMITS = ((0, -1.0, 0.7), (1, -1.2, 0.2), (3, -0.5, 1.0), (5, -0.9, 0.9))
HEIGHT_BOUNDS = ((0, 0.4, 0.9), (3, -0.1, 0.3))
N = 8


def main():
    ref_runner.import_cito()
    from dataclasses import replace

    from cito import ocp, scp

    import pyoracle
    from paper_2604_09993_b200.model import pack_model

    for mixing in ("identity", "ones"):
        t0 = time.time()
        sc = ocp.load_scenario(os.path.join(ref_runner.assets_dir(), "halfcheetah_bound.json"))
        sc = replace(sc, N=N, s_bounds=None, joint_angle_limits=JOINT_LIMITS, body_height_bounds=HEIGHT_BOUNDS,
                     mixing=mixing)
        tr = ocp.Transcription(sc)
        desc = pack_model(tr.model, tr.mixing, tr.path_fn)
        out = {"N": np.array(N), "substeps": np.array(sc.substeps), "mixing": np.array(mixing),
               "joint_limits": np.array(JOINT_LIMITS), "height_bounds": np.array(HEIGHT_BOUNDS)}

        def finite(x, u, s):  # redraw diverging draws (|end| > 1e6: chaotic, synth.well_posed)
            return synth.well_posed(pyoracle.propagate(desc, sc.substeps, x, u, s)[0])

        xt0, U, S, redrawn = synth.random_intervals(sc, 3, seed=3, finite_fn=finite)
        e, jx, ju, js = tr.discretizer.linearize_batch(xt0, U, S)
        out.update(lin_xt0=xt0, lin_U=U, lin_S=S, lin_ends=e, lin_jx=jx, lin_ju=ju, lin_js=js)
        print(mixing, "random linearize", time.time() - t0, flush=True)
        z = tr.initial_guess()
        lin = scp.linearize_all(tr, z, 1.0)
        out.update(ig_z=z, ig_ends=lin.ends, ig_jx=lin.jx, ig_ju=lin.ju, ig_js=lin.js, ig_defects=lin.defects,
                   ig_psi=lin.psi, ig_psi_jac=lin.psi_jac, ig_theta=lin.theta, ig_theta_jac=lin.theta_jac,
                   ig_imp=lin.imp_v, ig_imp_jac=lin.imp_jac)
        print(mixing, "linearize_all", time.time() - t0, flush=True)
        prog, meta = scp.build_subproblem(tr, lin, z, 1.0, scp.SCPConfig())
        out.update(sp0_A_indptr=prog.A.indptr, sp0_A_indices=prog.A.indices, sp0_A_data=prog.A.data,
                   sp0_A_shape=np.array(prog.A.shape), sp0_b=prog.b, sp0_G_indptr=prog.G.indptr,
                   sp0_G_indices=prog.G.indices, sp0_G_data=prog.G.data, sp0_G_shape=np.array(prog.G.shape),
                   sp0_h=prog.h, sp0_c=prog.c, sp0_nonneg=np.array(prog.cones.nonneg),
                   sp0_soc=np.array(prog.cones.soc))
        np.savez_compressed(os.path.join(HERE, f"halfcheetah_paths_{mixing}.npz"), **out)
        print(mixing, "done", prog.A.shape, prog.G.shape, time.time() - t0, flush=True)


if __name__ == "__main__":
    main()
