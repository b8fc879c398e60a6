"""Generate the golden fixtures from the UNMODIFIED reference (build container only).

Runs /root/reference/pkg/src/cito through oracle/ref_runner.py (jax -> torch.func
shim) and writes, per scenario, ``tests/golden/<name>.npz``:

  lin_*   Discretizer.linearize_batch on seeded synthetic intervals
          (paper_2604_09993_b200.synth)
  ig_*    linearize_all at the scenario's initial_guess() (SCP-realistic point):
          ends/jx/ju/js/defects + node relations and Jacobians
  nd_*    node_constraints/node_jacobians at a seeded random z (Phi != 0)
  csc_*   build_subproblem(...) -> canonicalize CSC of A/G (indptr, indices, data), b, h,
          at the initial guess, delta = 1 (cito/scp.py:160-351, cito/conic.py:209-269)

and copies the model/scenario JSON assets (data) to ``tests/golden/assets/`` so
the GPU box (no reference) can pose the same problems.

Usage:  python tests/golden/make_golden.py [name ...]
"""

import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import ref_runner  # noqa: E402

from paper_2604_09993_b200 import synth  # noqa: E402

# name -> (scenario file, N override or None, #random intervals, do CSC)
CASES = {
    "pointmass_rest": ("pointmass_rest", None, 4, True),
    "monoped_n20": ("monoped_hop", 20, 4, True),
    "halfcheetah_n30": ("halfcheetah_bound", 30, 4, True),
    "biped_walk": ("biped_walk", None, 3, True),
}


def main(names):
    cito = ref_runner.import_cito()
    from dataclasses import replace

    from cito import ocp, scp

    os.makedirs(os.path.join(HERE, "assets"), exist_ok=True)
    for f in os.listdir(ref_runner.assets_dir()):
        if f.endswith(".json"):
            shutil.copy(os.path.join(ref_runner.assets_dir(), f), os.path.join(HERE, "assets", f))

    for name in names:
        scen_name, N, n_rand, do_csc = CASES[name]
        t0 = time.time()
        sc = ocp.load_scenario(os.path.join(ref_runner.assets_dir(), scen_name + ".json"))
        if N is not None:
            sc = replace(sc, N=N, s_bounds=None)
        tr = ocp.Transcription(sc)
        lay = tr.layout
        out = {"scenario": np.array(scen_name), "N": np.array(sc.N), "substeps": np.array(sc.substeps)}

        # seeded synthetic intervals (uses the reference's own ScenarioSpec fields)
        import pyoracle
        from paper_2604_09993_b200.model import pack_model

        desc = pack_model(tr.model, tr.mixing, tr.path_fn)

        def finite(x, u, s):
            return pyoracle.propagate(desc, sc.substeps, x, u, s)[1] == 0

        xt0, U, S, redrawn = synth.random_intervals(sc, n_rand, seed=0, finite_fn=finite)
        out["lin_redrawn"] = np.array(redrawn)
        e, jx, ju, js = tr.discretizer.linearize_batch(xt0, U, S)
        out.update(lin_xt0=xt0, lin_U=U, lin_S=S, lin_ends=e, lin_jx=jx, lin_ju=ju, lin_js=js)
        print(name, "random linearize", time.time() - t0, flush=True)

        # SCP-realistic point: initial guess
        z = tr.initial_guess()
        delta = 1.0
        lin = scp.linearize_all(tr, z, delta)
        out.update(ig_z=z, ig_delta=np.array(delta), ig_eps=np.array(sc.ctcs_epsilon), ig_ends=lin.ends,
                   ig_jx=lin.jx, ig_ju=lin.ju, ig_js=lin.js, ig_defects=lin.defects, ig_psi=lin.psi,
                   ig_psi_jac=lin.psi_jac, ig_theta=lin.theta, ig_theta_jac=lin.theta_jac, ig_imp=lin.imp_v,
                   ig_imp_jac=lin.imp_jac)
        print(name, "initial-guess linearize_all", time.time() - t0, flush=True)

        # node relations at a random z (nonzero impulses)
        rng = np.random.default_rng(5)
        zr = 0.5 * rng.normal(size=lay.dim)
        nc = tr.node_constraints(zr, 0.05)
        pj, tj, ij = tr.node_jacobians(zr, 0.05)
        out.update(nd_z=zr, nd_delta=np.array(0.05), nd_psi=nc.psi, nd_theta=np.concatenate(
            [nc.theta_eq, nc.theta_ineq], axis=1), nd_imp=nc.impulse_defect[:, lay.n_q: 2 * lay.n_q],
            nd_psi_jac=pj, nd_theta_jac=tj, nd_imp_jac=ij)

        if do_csc:
            prog, meta = scp.build_subproblem(tr, lin, z, delta, scp.SCPConfig())
            out.update(csc_A_indptr=prog.A.indptr, csc_A_indices=prog.A.indices, csc_A_data=prog.A.data,
                       csc_A_shape=np.array(prog.A.shape), csc_b=prog.b, csc_G_indptr=prog.G.indptr,
                       csc_G_indices=prog.G.indices, csc_G_data=prog.G.data, csc_G_shape=np.array(prog.G.shape),
                       csc_h=prog.h, csc_n_dyn_rows=np.array((lay.N - 1) * lay.n_xt))
            print(name, "build_subproblem", time.time() - t0, flush=True)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, "done", time.time() - t0, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
