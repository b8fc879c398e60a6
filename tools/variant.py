"""A/B builds of the library restricted to a few topologies (fast: one template set).

  python tools/variant.py <name> [--topos halfcheetah_g2,...] [nvcc flags ...]

writes paper_2604_09993_b200/_lib/libcito_b200_<name>.so (load it with
CITO_LIB_VARIANT=<name>).  Kernel experiments only; the product build is build.py.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "paper_2604_09993_b200", "csrc"))

import gen_models  # noqa: E402

from paper_2604_09993_b200 import build as B  # noqa: E402
from paper_2604_09993_b200.topology import COMPILED  # noqa: E402


def main(argv):
    name = argv[0]
    topos = ["halfcheetah_g2"]
    flags = []
    it = iter(argv[1:])
    for a in it:
        if a == "--topos":
            topos = next(it).split(",")
        else:
            flags.append(a)
    entries = [e for e in COMPILED if e[0] in topos]
    out_dir = os.path.join(ROOT, "paper_2604_09993_b200", "_lib")
    hdr = os.path.join(out_dir, f"models_variant_{name}.cuh")
    gen_models.main(hdr, entries)
    so = os.path.join(out_dir, f"libcito_b200_{name}.so")
    cmd = [B.NVCC, "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler",
           "-fPIC", "-shared", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
           f'-DCITO_MODELS_GEN="{hdr}"', "-o", so] + flags + [os.path.join(B.CSRC, "cito_capi.cu"), "-lcudart"]
    subprocess.check_call(cmd)
    print(so)


if __name__ == "__main__":
    main(sys.argv[1:])
