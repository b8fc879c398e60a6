"""Drop-in test inside the reference's own SCP loop.

The unmodified reference package (installed copy in baseline/_ref, or
/root/reference in the build container) runs through the jax shim
(oracle/jaxshim, test infrastructure); its `cito.scp.linearize_all`,
`build_subproblem`, `precondition` and the transcription's discretizer are
replaced by the GPU implementations and
`cito.scp.solve` runs a few SCP iterations (host IPM + homotopy unchanged).
The iterates must match the reference's own path.  Runs in a subprocess so
the shim's global torch settings cannot leak into other tests.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_src():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "cito")):
            return p
    return None


SCRIPT = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.join(ROOT, "oracle"))
os.environ["CITO_REF_SRC"] = REF
sys.path.insert(0, ROOT)
import ref_runner
cito = ref_runner.import_cito()
from dataclasses import replace
from cito import ocp, scp
import paper_2604_09993_b200.linearize as G
import paper_2604_09993_b200.subproblem as SPB
from paper_2604_09993_b200 import install

name, iters, compare = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1"
sc = ocp.load_scenario(os.path.join(REF, "cito", "assets", name + ".json"))
cfg = scp.SCPConfig(max_iters=iters)
out = {}
if compare:
    ocp._transcriptions.clear()
    z_ref, hist_ref, st_ref = scp.solve(sc, cfg)
    out["ref"] = [h.z.tolist() for h in hist_ref]
    out["ref_delta"] = [h.delta for h in hist_ref]
ocp._transcriptions.clear()
tr = ocp.get_transcription(sc)
install(tr)                       # tr.discretizer -> GPU (initial_guess uses it)
orig = scp.linearize_all, scp.build_subproblem, scp.precondition
scp.linearize_all = G.linearize_all         # GPU linearize_all (intervals + node relations)
scp.build_subproblem = SPB.build_subproblem  # GPU subproblem assembly (CSC values, b, h)
scp.precondition = SPB.precondition          # GPU row scaling of the assembled program
try:
    z, hist, st = scp.solve(sc, cfg)
finally:
    scp.linearize_all, scp.build_subproblem, scp.precondition = orig
out["gpu"] = [h.z.tolist() for h in hist]
out["gpu_delta"] = [h.delta for h in hist]
out["status"] = st
out["launches"] = tr.discretizer.launch_count() + G._cache[id(tr)][1].disc.launch_count()
print("RESULT " + json.dumps(out))
'''


def _run(name, iters, compare, timeout=1500):
    ref = _ref_src()
    if ref is None:
        pytest.skip("reference package not available (baseline/_ref or /root/reference)")
    code = f"ROOT = {ROOT!r}\nREF = {ref!r}\n" + SCRIPT
    p = subprocess.run([sys.executable, "-c", code, name, str(iters), "1" if compare else "0"], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert p.returncode == 0 and line, p.stderr[-3000:]
    return json.loads(line[0][7:])


@pytest.mark.gpu
def test_scp_solve_pointmass_matches_reference_path():
    import numpy as np

    r = _run("pointmass_rest", 4, True)
    assert len(r["gpu"]) == len(r["ref"])
    for zg, zr in zip(r["gpu"], r["ref"]):
        zg, zr = np.asarray(zg), np.asarray(zr)
        assert np.max(np.abs(zg - zr)) <= 1e-6 * (1.0 + np.max(np.abs(zr)))
    assert np.allclose(r["gpu_delta"], r["ref_delta"], rtol=1e-9)
    assert r["launches"] > 0


@pytest.mark.gpu
def test_scp_solve_halfcheetah_runs_with_gpu_linearization():
    import numpy as np

    r = _run("halfcheetah_bound", 2, False)
    assert len(r["gpu"]) == 3
    assert all(np.all(np.isfinite(np.asarray(z))) for z in r["gpu"])
