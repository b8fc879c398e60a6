"""Build the sm_100a library in-tree: paper_2604_09993_b200/_lib/libcito_b200.so.

  python -m paper_2604_09993_b200.build [--force]

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, shared library
exporting the C ABI of include/cito_b200.h.  No GPU needed (cross-compile).
"""

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
DEPS = ["cito_capi.cu", "cito_kernels.cuh", "cito_k1v2.cuh", "cito_node.cuh", "cito_scatter.cuh", "cito_bench.cuh", "cito_subproblem.cuh", "gen_models.py"]


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, d) for d in DEPS]
    deps += [os.path.join(ROOT, "include", "cito_b200.h"), os.path.join(HERE, "topology.py")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return SO
    os.makedirs(OUT_DIR, exist_ok=True)
    subprocess.check_call([sys.executable, os.path.join(CSRC, "gen_models.py"),
                           os.path.join(CSRC, "models_gen.cuh")])
    cmd = [NVCC, "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-o", SO + ".tmp"]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    cmd += ["-lcudart"]
    subprocess.check_call(cmd)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
