"""Golden fixtures for the configs without reference parity in round 1 (build container only).

  halfcheetah_n200s8.npz   configs[4]: HalfCheetah N=200, 8 RKF substeps.
      ig_z       the reference's own Transcription.initial_guess() (unmodified
                 reference through the jax shim, oracle/ref_runner.py)
      ig_*       linearize_all at ig_z: the interval arrays (ends, jx, ju, js,
                 defects) by the pinned C oracle (the shim's jacfwd takes ~5 s per
                 interval; the oracle matches the reference's own linearization to
                 <= 1e-11, tests/test_oracle_golden.py), the node relations and
                 their Jacobians by the REFERENCE itself (Transcription.node_constraints /
                 node_jacobians, ~20 s): its LU leaves rounding residues (e.g.
                 2e-33 in imp_jac) where the oracle's elimination gives exact zeros,
                 and those residues are part of the CSC pattern
      sp0_*      the reference's build_subproblem -> canonicalize (cito/scp.py:160-351,
                 cito/conic.py:209-269) of that LinearizedProblem at delta = 1
      pcsp0_*    the reference's precondition (cito/conic.py:281-338) of sp0
      lin_*      4 seeded synthetic intervals linearized by the REFERENCE itself
                 (shim), pinning the oracle at 8 substeps

The sp0 values are a function of the oracle linearization, so the GPU assembler
fed with ig_* must reproduce them bit-exactly and the full GPU iteration within
rel 1e-9 with a bit-exact pattern.  N = 200 gives 3,904 CSC column blocks, more
than the B200 can hold resident, which is what the one-pass compaction's
look-back must survive.

Usage:  python tests/golden/make_golden_fine.py [--reuse]   (--reuse: keep ig_z and lin_* of the
        existing file, which the reference computed -- ~7 min through the shim)
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


def oracle_linearize_all(tr, desc, z, delta, substeps):
    """linearize_all (cito/scp.py:87-135) with the interval linearization of the pinned
    C oracle and the reference's own node relations; the gathers/defects follow
    scp.py:97-135."""
    import pyoracle

    from cito import scp

    lay = tr.layout
    N = lay.N
    starts = np.stack([z[lay.xp(k)] for k in range(N - 1)])
    Us = np.stack([z[lay.u(k)] for k in range(N - 1)])
    Ss = np.array([z[lay.s(k)][0] for k in range(N - 1)])
    e, jx, ju, js, bad = pyoracle.linearize(desc, substeps, starts, Us, Ss)
    assert not bad.any()
    defects = np.stack([z[lay.xm(k + 1)] for k in range(N - 1)]) - e
    nc = tr.node_constraints(z, delta)
    pj, tj, ij = tr.node_jacobians(z, delta)
    theta = np.concatenate([nc.theta_eq, nc.theta_ineq], axis=1)
    imp = nc.impulse_defect[:, lay.n_q: 2 * lay.n_q]
    return scp.LinearizedProblem(z_ref=z, ends=e, jx=jx, ju=ju, js=js, defects=defects, psi=nc.psi, psi_jac=pj,
                                 theta=theta, theta_jac=tj, imp_v=imp, imp_jac=ij)


def main():
    ref_runner.import_cito()
    from dataclasses import replace

    from cito import conic, ocp, scp

    import pyoracle
    from paper_2604_09993_b200.model import pack_model

    t0 = time.time()
    sc = ocp.load_scenario(os.path.join(ref_runner.assets_dir(), "halfcheetah_bound.json"))
    sc = replace(sc, N=200, substeps=8, s_bounds=None)
    tr = ocp.Transcription(sc)
    desc = pack_model(tr.model, tr.mixing, tr.path_fn)
    out = {"scenario": np.array("halfcheetah_bound"), "N": np.array(sc.N), "substeps": np.array(sc.substeps)}

    def finite(x, u, s):
        return pyoracle.propagate(desc, sc.substeps, x, u, s)[1] == 0

    path = os.path.join(HERE, "halfcheetah_n200s8.npz")
    old = dict(np.load(path)) if ("--reuse" in sys.argv and os.path.exists(path)) else None
    if old is not None:  # the reference-computed parts are deterministic: reuse them
        out.update({k: old[k] for k in old if k.startswith("lin_")})
        z = old["ig_z"]
    else:
        xt0, U, S, redrawn = synth.random_intervals(sc, 4, seed=0, finite_fn=finite)
        e, jx, ju, js = tr.discretizer.linearize_batch(xt0, U, S)
        out.update(lin_xt0=xt0, lin_U=U, lin_S=S, lin_ends=e, lin_jx=jx, lin_ju=ju, lin_js=js,
                   lin_redrawn=np.array(redrawn))
        print("reference linearize_batch (4 intervals, 8 substeps)", time.time() - t0, flush=True)
        z = tr.initial_guess()
        print("reference initial_guess", time.time() - t0, flush=True)
    lin = oracle_linearize_all(tr, desc, z, 1.0, sc.substeps)
    out.update(ig_z=z, ig_delta=np.array(1.0), ig_eps=np.array(sc.ctcs_epsilon), ig_ends=lin.ends, ig_jx=lin.jx,
               ig_ju=lin.ju, ig_js=lin.js, ig_defects=lin.defects, ig_psi=lin.psi, ig_psi_jac=lin.psi_jac,
               ig_theta=lin.theta, ig_theta_jac=lin.theta_jac, ig_imp=lin.imp_v, ig_imp_jac=lin.imp_jac)
    prog, meta = scp.build_subproblem(tr, lin, z, 1.0, scp.SCPConfig())
    print("reference build_subproblem", prog.A.shape, prog.A.nnz, prog.G.shape, prog.G.nnz, time.time() - t0,
          flush=True)
    tag = "sp0"
    out.update({f"{tag}_zj": z, f"{tag}_delta": np.array(1.0), f"{tag}_c": prog.c,
                f"{tag}_A_indptr": prog.A.indptr, f"{tag}_A_indices": prog.A.indices, f"{tag}_A_data": prog.A.data,
                f"{tag}_A_shape": np.array(prog.A.shape), f"{tag}_b": prog.b,
                f"{tag}_G_indptr": prog.G.indptr, f"{tag}_G_indices": prog.G.indices, f"{tag}_G_data": prog.G.data,
                f"{tag}_G_shape": np.array(prog.G.shape), f"{tag}_h": prog.h,
                f"{tag}_nonneg": np.array(prog.cones.nonneg), f"{tag}_soc": np.array(prog.cones.soc)})
    out.update({f"{tag}_P_indptr": prog.P.indptr, f"{tag}_P_indices": prog.P.indices, f"{tag}_P_data": prog.P.data})
    scaled, prec = conic.precondition(prog)
    out.update({f"pc{tag}_A_data": scaled.A.data, f"pc{tag}_G_data": scaled.G.data, f"pc{tag}_b": scaled.b,
                f"pc{tag}_h": scaled.h, f"pc{tag}_c": scaled.c, f"pc{tag}_P_data": scaled.P.data,
                f"pc{tag}_row_scale_A": prec.row_scale_A, f"pc{tag}_row_scale_G": prec.row_scale_G,
                f"pc{tag}_cost_scale": np.array(prec.cost_scale)})
    np.savez_compressed(path, **out)
    print("done", time.time() - t0, flush=True)


if __name__ == "__main__":
    main()
