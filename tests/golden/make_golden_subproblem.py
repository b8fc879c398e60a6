"""Add the reference's full subproblem (P, c, A, b, G, h, cones) to the golden files.

Rebuilds `cito.scp.build_subproblem` (unmodified reference, via oracle/ref_runner.py)
from the LinearizedProblem already stored in tests/golden/<name>.npz (ig_*), at
the initial guess (delta = 1) and at a second, perturbed iterate z_j with
delta = 0.3 (same linearization), so the tests cover both pattern variants.
Writes sp0_* / sp1_* arrays into the same npz.  Build container only.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref_runner  # noqa: E402

CASES = {"pointmass_rest": ("pointmass_rest", None), "monoped_n20": ("monoped_hop", 20),
         "halfcheetah_n30": ("halfcheetah_bound", 30), "biped_walk": ("biped_walk", None)}


def main(names):
    ref_runner.import_cito()
    from dataclasses import replace

    from cito import ocp, scp

    for name in names:
        scen, N = CASES[name]
        path = os.path.join(HERE, name + ".npz")
        g = dict(np.load(path))
        sc = ocp.load_scenario(os.path.join(ref_runner.assets_dir(), scen + ".json"))
        if N is not None:
            sc = replace(sc, N=N, s_bounds=None)
        tr = ocp.Transcription(sc)
        lin = scp.LinearizedProblem(z_ref=g["ig_z"], ends=g["ig_ends"], jx=g["ig_jx"], ju=g["ig_ju"], js=g["ig_js"],
                                    defects=g["ig_defects"], psi=g["ig_psi"], psi_jac=g["ig_psi_jac"],
                                    theta=g["ig_theta"], theta_jac=g["ig_theta_jac"], imp_v=g["ig_imp"],
                                    imp_jac=g["ig_imp_jac"])
        rng = np.random.default_rng(9)
        zj1 = g["ig_z"] + 0.01 * rng.normal(size=g["ig_z"].size)
        # sp2: node relations at a random z with nonzero impulses (nd_*), which moves the
        # node-row pattern; interval arrays reused, z_ref = that z
        lin2 = scp.LinearizedProblem(z_ref=g["nd_z"], ends=g["ig_ends"], jx=g["ig_jx"], ju=g["ig_ju"], js=g["ig_js"],
                                     defects=g["ig_defects"], psi=g["nd_psi"], psi_jac=g["nd_psi_jac"],
                                     theta=g["nd_theta"], theta_jac=g["nd_theta_jac"], imp_v=g["nd_imp"],
                                     imp_jac=g["nd_imp_jac"])
        for tag, zj, delta, ln in (("sp0", g["ig_z"], 1.0, lin), ("sp1", zj1, 0.3, lin), ("sp2", g["nd_z"], 0.05, lin2)):
            prog, meta = scp.build_subproblem(tr, ln, zj, delta, scp.SCPConfig())
            g.update({f"{tag}_zj": zj, f"{tag}_delta": np.array(delta),
                      f"{tag}_P_indptr": prog.P.indptr, f"{tag}_P_indices": prog.P.indices,
                      f"{tag}_P_data": prog.P.data, f"{tag}_c": prog.c,
                      f"{tag}_A_indptr": prog.A.indptr, f"{tag}_A_indices": prog.A.indices,
                      f"{tag}_A_data": prog.A.data, f"{tag}_A_shape": np.array(prog.A.shape), f"{tag}_b": prog.b,
                      f"{tag}_G_indptr": prog.G.indptr, f"{tag}_G_indices": prog.G.indices,
                      f"{tag}_G_data": prog.G.data, f"{tag}_G_shape": np.array(prog.G.shape), f"{tag}_h": prog.h,
                      f"{tag}_nonneg": np.array(prog.cones.nonneg), f"{tag}_soc": np.array(prog.cones.soc)})
            print(name, tag, prog.A.shape, prog.A.nnz, prog.G.shape, prog.G.nnz, flush=True)
        np.savez_compressed(path, **g)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
