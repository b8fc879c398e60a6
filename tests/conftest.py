import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # test infrastructure: the CPU oracle

GOLDEN = os.path.join(ROOT, "tests", "golden")
GOLDEN_CASES = ["pointmass_rest", "monoped_n20", "halfcheetah_n30", "biped_walk"]
SCEN_OF = {"pointmass_rest": ("pointmass_rest", {}), "monoped_n20": ("monoped_hop", {"N": 20}),
           "halfcheetah_n30": ("halfcheetah_bound", {"N": 30}), "biped_walk": ("biped_walk", {}),
           "halfcheetah_n200s8": ("halfcheetah_bound", {"N": 200, "substeps": 8})}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def rel_err(a, b):
    """max|a-b| / (1 + max|b|): the reference's own _rel_err (tests/test_acceptance.py:168-169)."""
    a, b = np.asarray(a), np.asarray(b)
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))))


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def golden_scenario(name):
    from paper_2604_09993_b200 import scenario as S

    scen, overrides = SCEN_OF[name]
    return S.bundled(scen, **overrides)


def scenario_desc(sc):
    from paper_2604_09993_b200.model import pack_model

    g, n_g = sc.path_constraints()
    return pack_model(sc.model, sc.mixing_matrix(n_g), g)


@pytest.fixture(params=GOLDEN_CASES)
def golden_case(request):
    name = request.param
    return name, load_golden(name), golden_scenario(name)


def pytest_sessionstart(session):
    # the product library and the oracle are built in-tree (no-ops when fresh)
    from paper_2604_09993_b200 import build

    build.build()
    import pyoracle

    pyoracle.build()
