"""Add the reference's replay audit (cito.verifier.replay_check) to the golden files.

Runs the UNMODIFIED reference `replay_check(z, model, scenario, grid)`
(verifier.py:236-346, via oracle/ref_runner.py and the jax shim) at the stored
initial-guess decision vector ig_z (and, for the small cases, at the random
node point nd_z) and stores rp{tag}_* = every FeasibilityReport field.
Build container only (reads /root/reference).  The shim integrates in eager
torch, so this takes minutes for HalfCheetah.

Usage:  python tests/golden/make_golden_replay.py [name ...]
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref_runner  # noqa: E402

# name -> (scenario, N override, grid, z tags)
CASES = {"pointmass_rest": ("pointmass_rest", None, 20, ("ig", "nd")),
         "monoped_n20": ("monoped_hop", 20, 8, ("ig",)),
         "halfcheetah_n30": ("halfcheetah_bound", 30, 4, ("ig",))}


def main(names):
    ref_runner.import_cito()
    from dataclasses import replace

    from cito import ocp, verifier

    for name in names:
        scen, N, grid, tags = CASES[name]
        path = os.path.join(HERE, name + ".npz")
        g = dict(np.load(path))
        sc = ocp.load_scenario(os.path.join(ref_runner.assets_dir(), scen + ".json"))
        if N is not None:
            sc = replace(sc, N=N, s_bounds=None)
        tr = ocp.get_transcription(sc)
        for tag in tags:
            t0 = time.time()
            rep = verifier.replay_check(g[f"{tag}_z"], tr.model, sc, grid=grid)
            g.update({f"rp{tag}_grid": np.array(grid), f"rp{tag}_max_penetration": np.array(rep.max_penetration),
                      f"rp{tag}_max_joint_drift": np.array(rep.max_joint_drift),
                      f"rp{tag}_pair_residuals": rep.pair_residuals, f"rp{tag}_ctcs_increments": rep.ctcs_increments,
                      f"rp{tag}_ctcs_epsilon": np.array(rep.ctcs_epsilon),
                      f"rp{tag}_cone_violation": np.array(rep.cone_violation),
                      f"rp{tag}_refinement_drift": np.array(rep.refinement_drift),
                      f"rp{tag}_cross_products": rep.cross_products})
            print(name, tag, f"{time.time() - t0:.1f}s", rep.max_penetration, rep.max_joint_drift,
                  rep.refinement_drift, rep.cone_violation, float(np.max(rep.cross_products)), flush=True)
        np.savez_compressed(path, **g)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
