"""Build the sm_100a library in-tree: paper_2604_09993_b200/_lib/libcito_b200.so.

  python -m paper_2604_09993_b200.build [--force]

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, shared library
exporting the C ABI of include/cito_b200.h.  No GPU needed (cross-compile).

The bundled library carries the topologies of topology.COMPILED.  Any other
RobotModel topology (within the kernel limits) is compiled on first use by
``build_topology``: the same sources with a one-entry topology table
(-DCITO_MODELS_GEN), into _lib/jit/libcito_b200_<name>.so, cached by the
topology key -- the analogue of the reference jitting its closures per model
(cito/augmentation.py:180-216).
"""

import fcntl
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
SO = os.path.join(OUT_DIR, "libcito_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["cito_capi.cu"]
DEPS = ["cito_capi.cu", "cito_kernels.cuh", "cito_k1v2.cuh", "cito_node.cuh", "cito_scatter.cuh", "cito_bench.cuh",
        "cito_subproblem.cuh", "gen_models.py"]


def _deps():
    deps = [os.path.join(CSRC, d) for d in DEPS]
    return deps + [os.path.join(ROOT, "include", "cito_b200.h"), os.path.join(HERE, "topology.py")]


def _stale(so):
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(d) > t for d in _deps())


def _nvcc(out, defines=(), verbose=False):
    cmd = [NVCC, "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp"] + list(defines)
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    cmd += ["-lcudart"]
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)


def build(force=False, verbose=False):
    if not force and not _stale(SO):
        return SO
    os.makedirs(OUT_DIR, exist_ok=True)
    subprocess.check_call([sys.executable, os.path.join(CSRC, "gen_models.py"),
                           os.path.join(CSRC, "models_gen.cuh")])
    _nvcc(SO, verbose=verbose)
    return SO


def jit_dir():
    return os.environ.get("CITO_JIT_DIR", os.path.join(OUT_DIR, "jit"))


def build_topology(entry, force=False):
    """Compile a library whose topology table holds only `entry` (a
    topology.COMPILED-style tuple, see topology.entry_from_desc).  Returns the
    path of the shared library; concurrent builders of the same topology
    serialise on a lock file."""
    sys.path.insert(0, CSRC)
    import gen_models

    name = entry[0]
    d = jit_dir()
    os.makedirs(d, exist_ok=True)
    so = os.path.join(d, f"libcito_b200_{name}.so")
    with open(os.path.join(d, f".{name}.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if force or _stale(so):
            hdr = os.path.join(d, f"models_{name}.cuh")
            gen_models.main(hdr, [entry])
            _nvcc(so, defines=[f'-DCITO_MODELS_GEN="{hdr}"'])
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
