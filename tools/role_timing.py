"""Per-role cycle timing of the fused linearize kernel (CTA 0), via a -DCITO_PROF build.

  python tools/role_timing.py build          # (CPU) build paper_2604_09993_b200/_lib/libcito_b200_prof.so
  python tools/role_timing.py run [B]        # (GPU) print per-tick cycles of each warp role
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROF_SO = os.path.join(ROOT, "paper_2604_09993_b200", "_lib", "libcito_b200_prof.so")


def build(extra=()):
    # HalfCheetah-only variant library (tools/variant.py) with the cycle marks compiled in
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "variant.py"), "prof", "-DCITO_PROF",
                           *extra])


def run(B):
    import ctypes

    import numpy as np
    import torch

    from paper_2604_09993_b200 import _lib

    _lib.SO_PATH = PROF_SO
    from paper_2604_09993_b200 import scenario as S, synth, Discretizer

    L = _lib.lib()
    L.cito_prof_set.argtypes = [ctypes.c_void_p]
    sc = S.bundled("halfcheetah_bound", N=30)
    g, n_g = sc.path_constraints()
    disc = Discretizer(sc.model, sc.mixing_matrix(n_g), g, substeps=sc.substeps)
    x, U, Sv = synth.random_intervals(sc, B, seed=0)
    dev = torch.device("cuda")
    xd, Ud, Sd = (torch.as_tensor(a, device=dev) for a in (x, U, Sv))
    buf = torch.zeros(1024 + 40 * 16 + 16, dtype=torch.int64, device=dev)
    for _ in range(3):
        disc.linearize_batch_device(xd, Ud, Sd)
    torch.cuda.synchronize()
    assert L.cito_prof_set(buf.data_ptr()) == 0
    disc.linearize_batch_device(xd, Ud, Sd)
    torch.cuda.synchronize()
    L.cito_prof_set(None)
    full = buf.cpu().numpy().astype(np.int64)
    a = full[:640].reshape(40, 8, 2)
    pp = full[1024:1024 + 640].reshape(40, 16)
    for t in (3, 10, 17):
        row = pp[t][pp[t] > 0]
        print("primal tick", t, "sub-step cycles", np.diff(row).tolist())
    nt = 32
    t0 = a[0, :, 0][a[0, :, 0] > 0].min()
    nw = int(sum(1 for w in range(8) if a[2, w, 0] > 0))
    print("tick  " + "  ".join(f"w{w}:work" for w in range(nw)) + "   tick_total")
    tot = []
    for t in range(nt):
        st, en = a[t, :nw, 0], a[t, :nw, 1]
        if not (st > 0).all():
            continue
        nxt = a[t + 1, :nw, 0].min() if t + 1 < nt and (a[t + 1, :nw, 0] > 0).all() else en.max()
        tot.append(nxt - st.min())
        print(f"{t:4d}  " + "  ".join(f"{int(e - s):8d}" for s, e in zip(st, en)) + f"   {int(nxt - st.min()):8d}")
    print("total cycles", int(a[nt - 1, :nw, 1].max() - t0), "mean tick", float(np.mean(tot)))
    k0, k1 = int(full[1664]), int(full[1665])
    if k0 and k1:
        print("kernel (CTA 0) cycles", k1 - k0, "prologue", int(t0 - k0),
              "after tick", nt - 1, int(k1 - a[nt - 1, :nw, 1].max()), "(the remaining ticks + outputs)")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(int(sys.argv[2]) if len(sys.argv) > 2 else 29)
