"""Algorithmic FLOPs per interval linearization -> profiles/flops_per_interval.json.

Counted by the instrumented C oracle (oracle_count_flops): the flops a
structurally sparse forward mode executes over the reference's discrete RKF
recursion (value flop + work on nonzero tangent entries only; + - * / sqrt sin
cos = 1, FMA = 2), SURVEY.md §8(d).  Median over 16 seeded synthetic intervals.
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402

from paper_2604_09993_b200 import scenario as S, synth  # noqa: E402
from paper_2604_09993_b200.model import pack_model  # noqa: E402

CASES = {
    "halfcheetah_s5": ("halfcheetah_bound", dict(N=30)),
    "halfcheetah_s8": ("halfcheetah_bound", dict(N=200, substeps=8)),
    "halfcheetah_s10": ("halfcheetah_bound", dict(N=30, substeps=10)),
    "monoped_s10": ("monoped_hop", dict(N=20)),
    "biped_s5": ("biped_walk", {}),
}


def main():
    out = {"definition": "structurally-sparse forward-mode flops of one interval linearization (ends + "
                         "Phi + B- + B+ + dS) of the reference's RKF recursion; +,-,*,/,sqrt,sin,cos = 1, "
                         "FMA = 2; counted by oracle_count_flops (oracle/cito_oracle.c)"}
    for key, (name, ov) in CASES.items():
        sc = S.bundled(name, **ov)
        g, n_g = sc.path_constraints()
        d = pack_model(sc.model, sc.mixing_matrix(n_g), g)
        x, U, Sv = synth.random_intervals(sc, 16, seed=0)
        f = [pyoracle.count_flops(d, sc.substeps, x[i], U[i], Sv[i]) for i in range(16)]
        out[key] = {"scenario": name, "overrides": ov, "substeps": sc.substeps, "flops": float(np.median(f)),
                    "min": float(min(f)), "max": float(max(f))}
        print(key, out[key])
    with open(os.path.join(ROOT, "profiles", "flops_per_interval.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
