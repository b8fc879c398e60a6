import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import pyoracle
from conftest import golden_scenario, scenario_desc, rel_err
from paper_2604_09993_b200 import synth, Discretizer
sc = golden_scenario("biped_walk"); desc = scenario_desc(sc)
g, n_g = sc.path_constraints()
disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
xt0, U, S, _ = synth.random_intervals(sc, 96, seed=11, finite_fn=lambda x, u, s: pyoracle.propagate(desc, sc.substeps, x, u, s)[1] == 0)
ref = pyoracle.linearize(desc, sc.substeps, xt0, U, S)
out = disc.linearize_batch(xt0, U, S)
names = ["ends", "jx", "ju", "js"]
for b in range(96):
    errs = [rel_err(a[b], r[b]) for a, r in zip(out, ref[:4])]
    if max(errs) > 1e-9:
        print(b, ["%s %.2e" % (n, e) for n, e in zip(names, errs)], "max|ref|", [float(np.abs(r[b]).max()) for r in ref[:4]])
        d = np.abs(out[1][b] - ref[1][b]); i, j = np.unravel_index(d.argmax(), d.shape)
        print("   jx worst at", i, j, out[1][b][i, j], ref[1][b][i, j])
        d = np.abs(out[0][b] - ref[0][b]); print("   ends worst", d.argmax(), out[0][b][d.argmax()], ref[0][b][d.argmax()])
