"""ctypes wrapper of the C oracle (TEST INFRASTRUCTURE ONLY).

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU legs, as
the checker / CPU baseline.  Builds ``_build/libcito_oracle.so`` on demand.
"""

import ctypes
import os
import subprocess

import numpy as np



_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libcito_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)


def build():
    src = os.path.join(_HERE, "cito_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.oracle_linearize.restype = ctypes.c_int
        L.oracle_linearize.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, _dp, _dp, _dp, _dp,
                                       _dp, _dp, _dp, _ip]
        L.oracle_propagate.restype = ctypes.c_int
        L.oracle_propagate.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, _dp, _dp, _dp, _dp, _ip]
        L.oracle_node_linearize.restype = None
        L.oracle_node_linearize.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, _dp, _dp,
                                            ctypes.c_double, ctypes.c_double, _dp, _dp, _dp, _dp, _dp, _dp]
        L.oracle_count_flops.restype = ctypes.c_double
        L.oracle_count_flops.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp, ctypes.c_double]
        L.oracle_set_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp)


def _dims(desc):
    nq = 3 * desc.n_links
    na = sum(1 for j in range(desc.n_joints) if desc.joint_actuated[j])
    nu = na + 3 * desc.n_contacts
    ny = 5 * desc.n_contacts + desc.n_g_out
    return nq, nu, ny, 2 * nq + ny


def linearize(desc, substeps, xt0s, Us, Ss):
    nq, nu, ny, nxt = _dims(desc)
    xt0s = np.ascontiguousarray(xt0s, dtype=np.float64).reshape(-1, nxt)
    B = xt0s.shape[0]
    Us = np.ascontiguousarray(Us, dtype=np.float64).reshape(B, 2 * nu)
    Ss = np.ascontiguousarray(Ss, dtype=np.float64).reshape(B)
    ends = np.empty((B, nxt))
    jx = np.empty((B, nxt, nxt))
    ju = np.empty((B, nxt, 2 * nu))
    js = np.empty((B, nxt))
    bad = np.zeros(B, dtype=np.int32)
    lib().oracle_linearize(ctypes.byref(desc), int(substeps), B, _p(xt0s), _p(Us), _p(Ss), _p(ends), _p(jx),
                           _p(ju), _p(js), bad.ctypes.data_as(_ip))
    return ends, jx, ju, js, bad


def propagate(desc, substeps, xt0s, Us, Ss):
    nq, nu, ny, nxt = _dims(desc)
    xt0s = np.ascontiguousarray(xt0s, dtype=np.float64).reshape(-1, nxt)
    B = xt0s.shape[0]
    Us = np.ascontiguousarray(Us, dtype=np.float64).reshape(B, 2 * nu)
    Ss = np.ascontiguousarray(Ss, dtype=np.float64).reshape(B)
    ends = np.empty((B, nxt))
    bad = np.zeros(B, dtype=np.int32)
    lib().oracle_propagate(ctypes.byref(desc), int(substeps), B, _p(xt0s), _p(Us), _p(Ss), _p(ends),
                           bad.ctypes.data_as(_ip))
    return ends, bad


def node_linearize(desc, y_pairs, theta_vecs, delta, epsilon):
    nq, nu, ny, nxt = _dims(desc)
    nc = desc.n_contacts
    npsi = 3 * nc + desc.n_g_out
    y_pairs = np.ascontiguousarray(y_pairs, dtype=np.float64).reshape(-1, 2 * ny)
    theta_vecs = np.ascontiguousarray(theta_vecs, dtype=np.float64).reshape(-1, 3 * nq + 3 * nc)
    Np, Nn = y_pairs.shape[0], theta_vecs.shape[0]
    psi = np.empty((Np, npsi))
    psi_jac = np.empty((Np, npsi, 2 * ny))
    th = np.empty((Nn, 6 * nc))
    th_jac = np.empty((Nn, 6 * nc, 3 * nq + 3 * nc))
    imp = np.empty((Nn, nq))
    imp_jac = np.empty((Nn, nq, 3 * nq + 2 * nc))
    lib().oracle_node_linearize(ctypes.byref(desc), Np, Nn, _p(y_pairs), _p(theta_vecs), float(delta),
                                float(epsilon), _p(psi), _p(psi_jac), _p(th), _p(th_jac), _p(imp),
                                _p(imp_jac))
    return psi, psi_jac, th, th_jac, imp, imp_jac


def count_flops(desc, substeps, xt0, U, S):
    """Structurally-sparse forward-mode flops of one interval linearization."""
    xt0 = np.ascontiguousarray(xt0, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64).reshape(-1)
    if U.size == 0:
        U = np.zeros(1)
    return float(lib().oracle_count_flops(ctypes.byref(desc), int(substeps), _p(xt0), _p(U), float(S)))


def set_threads(n):
    return lib().oracle_set_threads(int(n))


def get_threads():
    return lib().oracle_get_threads()
