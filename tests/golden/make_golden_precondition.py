"""Add the reference's preconditioned subproblem to the golden files.

For every sp0/sp1/sp2 program already stored in tests/golden/<name>.npz (the
reference's own build_subproblem output, make_golden_subproblem.py), run the
UNMODIFIED `cito.conic.precondition` (conic.py:290-338, via oracle/ref_runner.py)
and store pc{tag}_* = scaled A/G data, b, h, c, P data, row_scale_A/G, cost_scale.
Build container only (reads /root/reference).

Usage:  python tests/golden/make_golden_precondition.py [name ...]
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref_runner  # noqa: E402

CASES = ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]
TAGS = ["sp0", "sp1", "sp2"]


def program(conic, g, tag):
    n = int(g[f"{tag}_A_shape"][1])
    mat = lambda M: sp.csc_matrix((g[f"{tag}_{M}_data"], g[f"{tag}_{M}_indices"], g[f"{tag}_{M}_indptr"]),  # noqa: E731
                                  shape=tuple(g[f"{tag}_{M}_shape"]))
    P = sp.csc_matrix((g[f"{tag}_P_data"], g[f"{tag}_P_indices"], g[f"{tag}_P_indptr"]), shape=(n, n))
    cones = conic.ConeSpec(nonneg=int(g[f"{tag}_nonneg"]), soc=tuple(int(d) for d in g[f"{tag}_soc"]))
    return conic.ConicProgram(P=P, c=g[f"{tag}_c"], A=mat("A"), b=g[f"{tag}_b"], G=mat("G"), h=g[f"{tag}_h"],
                              cones=cones)


def main(names):
    ref_runner.import_cito()
    from cito import conic

    for name in names:
        path = os.path.join(HERE, name + ".npz")
        g = dict(np.load(path))
        for tag in TAGS:
            scaled, prec = conic.precondition(program(conic, g, tag))
            for M in ("A", "G"):
                M_s = getattr(scaled, M)
                assert np.array_equal(M_s.indptr, g[f"{tag}_{M}_indptr"]) and np.array_equal(
                    M_s.indices, g[f"{tag}_{M}_indices"]), "precondition must keep the pattern"
            g.update({f"pc{tag}_A_data": scaled.A.data, f"pc{tag}_G_data": scaled.G.data, f"pc{tag}_b": scaled.b,
                      f"pc{tag}_h": scaled.h, f"pc{tag}_c": scaled.c, f"pc{tag}_P_data": scaled.P.data,
                      f"pc{tag}_row_scale_A": prec.row_scale_A, f"pc{tag}_row_scale_G": prec.row_scale_G,
                      f"pc{tag}_cost_scale": np.array(prec.cost_scale)})
            print(name, tag, "cost_scale", prec.cost_scale, "min row scale A/G",
                  prec.row_scale_A.min(), prec.row_scale_G.min(), flush=True)
        np.savez_compressed(path, **g)


if __name__ == "__main__":
    main(sys.argv[1:] or CASES)
