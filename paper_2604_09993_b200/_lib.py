"""ctypes binding of libcito_b200.so (the C ABI of include/cito_b200.h).

There is no CPU fallback: if the library is missing this module raises at
import, and every compute entry point requires a CUDA device.
"""

import ctypes
import os
import threading

from .model import Dims, ModelDesc

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "_lib", "libcito_b200.so")
# A/B builds of the same library for kernel experiments (tools/ only); in-tree like the product library
if os.environ.get("CITO_LIB_VARIANT"):
    SO_PATH = os.path.join(_HERE, "_lib", f"libcito_b200_{os.environ['CITO_LIB_VARIANT']}.so")

CITO_OK, CITO_ERR_ARG, CITO_ERR_NONFINITE, CITO_ERR_CUDA, CITO_ERR_UNSUPPORTED = range(5)

_dp = ctypes.c_void_p  # device or host double* (raw address)
_lock = threading.Lock()
_lib = None


class CitoError(RuntimeError):
    pass


class UnsupportedModelError(CitoError, NotImplementedError):
    pass


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH):
            raise ImportError(
                f"{SO_PATH} not built; run `python -m paper_2604_09993_b200.build` "
                "(there is no CPU fallback for the discretize/linearize path)")
        _lib = _configure(ctypes.CDLL(SO_PATH))
        return _lib


def _configure(L):
    L.cito_last_error.restype = ctypes.c_char_p
    L.cito_version.restype = ctypes.c_char_p
    L.cito_create.restype = ctypes.c_int
    L.cito_create.argtypes = [ctypes.POINTER(ModelDesc), ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
    L.cito_destroy.restype = ctypes.c_int
    L.cito_destroy.argtypes = [ctypes.c_void_p]
    L.cito_get_dims.restype = ctypes.c_int
    L.cito_get_dims.argtypes = [ctypes.c_void_p, ctypes.POINTER(Dims)]
    L.cito_launch_count.restype = ctypes.c_int64
    L.cito_launch_count.argtypes = [ctypes.c_void_p]
    L.cito_linearize_host.restype = ctypes.c_int
    L.cito_linearize_host.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [_dp] * 8
    L.cito_linearize_dev.restype = ctypes.c_int
    L.cito_linearize_dev.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [_dp] * 9
    L.cito_propagate_host.restype = ctypes.c_int
    L.cito_propagate_host.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [_dp] * 5
    L.cito_propagate_dev.restype = ctypes.c_int
    L.cito_propagate_dev.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [_dp] * 6
    L.cito_node_linearize_dev.restype = ctypes.c_int
    L.cito_node_linearize_dev.argtypes = ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, _dp, _dp,
                                           ctypes.c_double, ctypes.c_double] + [_dp] * 7)
    L.cito_scatter_dynamics_dev.restype = ctypes.c_int
    L.cito_scatter_dynamics_dev.argtypes = ([ctypes.c_void_p, ctypes.c_int64] + [_dp] * 10 +
                                            [ctypes.c_double] + [_dp] * 7)
    L.cito_linearize_all_dev.restype = ctypes.c_int
    L.cito_linearize_all_dev.argtypes = ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int64, _dp, ctypes.c_double, ctypes.c_double]
                                         + [_dp] * 13)
    L.cito_audit_dev.restype = ctypes.c_int
    L.cito_audit_dev.argtypes = [ctypes.c_void_p, ctypes.c_int64, _dp, ctypes.c_int64] + [_dp] * 5
    L.cito_linearize_all_dev2.restype = ctypes.c_int
    L.cito_linearize_all_dev2.argtypes = ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int64, _dp, _dp] + [_dp] * 13)
    L.cito_csc_assemble_dev.restype = ctypes.c_int
    L.cito_csc_assemble_dev.argtypes = [ctypes.c_int32] + [_dp] * 12
    L.cito_csc_assemble2_dev.restype = ctypes.c_int
    L.cito_csc_assemble2_dev.argtypes = [ctypes.c_int32, ctypes.c_int32] + [_dp] * 13
    L.cito_precondition_dev.restype = ctypes.c_int
    L.cito_precondition_dev.argtypes = ([ctypes.c_int32] + [_dp] * 3 + [ctypes.c_int32, _dp] + [_dp] * 3 +
                                        [ctypes.c_int32, _dp, ctypes.c_int32, ctypes.c_int32] + [_dp] * 4 +
                                        [ctypes.c_int32, ctypes.c_int32] + [_dp] * 6 + [ctypes.c_int64, _dp])
    L.cito_csc_assemble_packed_dev.restype = ctypes.c_int
    L.cito_csc_assemble_packed_dev.argtypes = ([ctypes.c_int32, ctypes.c_int32] + [_dp] * 7 + [ctypes.c_int64] +
                                               [_dp] * 6 + [ctypes.c_int64, ctypes.c_int64, _dp, _dp, _dp])
    L.cito_copy_mirror.restype = ctypes.c_int
    L.cito_copy_mirror.argtypes = [_dp, _dp, ctypes.c_int64, ctypes.c_int64, _dp]
    L.cito_rhs_dev.restype = ctypes.c_int
    L.cito_rhs_dev.argtypes = [ctypes.c_int64] + [_dp] * 12 + [ctypes.c_int64, _dp]
    L.cito_dfma_peak.restype = ctypes.c_double
    L.cito_dfma_peak.argtypes = [ctypes.c_int32, _dp, _dp]
    return L


def lib():
    return _load()


_jit_libs = {}  # topology key -> CDLL of a run-time compiled single-topology library


def lib_for_topology(desc):
    """The library that carries the topology of `desc`: compiled on first use
    (build.build_topology, ~20 s of nvcc) when the bundled one does not.
    CITO_JIT=0 turns the run-time build off (UnsupportedModelError instead)."""
    from . import build as _build
    from .topology import entry_from_desc

    entry, key = entry_from_desc(desc)
    with _lock:
        L = _jit_libs.get(key)
        if L is not None:
            return L
    if os.environ.get("CITO_JIT", "1") == "0":
        raise UnsupportedModelError(f"model topology {key} is not in the bundled library and CITO_JIT=0")
    so = _build.build_topology(entry)
    with _lock:
        L = _jit_libs.get(key)
        if L is None:
            L = _jit_libs[key] = _configure(ctypes.CDLL(so))
    return L


def loaded_libraries():
    libs = [lib()]
    with _lock:
        libs += list(_jit_libs.values())
    return libs


_graph_launches = 0  # library kernels launched through CUDA-graph replays (not seen by the C counter)


def add_graph_launches(n):
    global _graph_launches
    _graph_launches += int(n)


def launch_count():
    """Kernels of this library launched so far (every loaded copy: the bundled one and
    run-time compiled topologies): direct launches (C counters) + graph replays."""
    return sum(int(L.cito_launch_count(None)) for L in loaded_libraries()) + _graph_launches


def check(status, what="", L=None):
    if status == CITO_OK:
        return
    msg = (L or lib()).cito_last_error().decode(errors="replace")
    if status == CITO_ERR_NONFINITE:
        raise FloatingPointError(msg)
    if status == CITO_ERR_ARG:
        raise ValueError(msg)
    if status == CITO_ERR_UNSUPPORTED:
        raise UnsupportedModelError(msg)
    raise CitoError(f"{what}: {msg}")


class Handle:
    """Owns one cito_handle (per model/mixing/path spec/substeps)."""

    def __init__(self, desc, substeps):
        self._ptr = ctypes.c_void_p()
        self.desc = desc
        L = lib()
        st = L.cito_create(ctypes.byref(desc), int(substeps), ctypes.byref(self._ptr))
        if st == CITO_ERR_UNSUPPORTED:  # topology outside the bundled set: run-time compiled library
            L = lib_for_topology(desc)
            st = L.cito_create(ctypes.byref(desc), int(substeps), ctypes.byref(self._ptr))
        self.L = L  # every entry point taking this handle must be called on its own library
        check(st, "cito_create", L)
        d = Dims()
        check(L.cito_get_dims(self._ptr, ctypes.byref(d)), "cito_get_dims", L)
        self.dims = d

    @property
    def ptr(self):
        return self._ptr

    def launch_count(self):
        return int(self.L.cito_launch_count(self._ptr))

    def check(self, status, what=""):
        check(status, what, self.L)

    def __del__(self):
        try:
            if self._ptr:
                self.L.cito_destroy(self._ptr)
                self._ptr = ctypes.c_void_p()
        except Exception:
            pass


def addr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
