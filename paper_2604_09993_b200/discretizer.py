"""Drop-in replacement of ``cito.augmentation.Discretizer`` backed by sm_100a kernels.

Same constructor, attributes, methods, outputs and error behaviour as the
reference class (/root/reference/pkg/src/cito/augmentation.py:172-255):

  Discretizer(model, mixing=None, path_fn=None, substeps=10)   ValueError if substeps < 1
  .model .mixing .path_fn .substeps .n_y .n_xt
  .propagate(xt0, U, S) -> (n_xt,)            FloatingPointError on non-finite end
  .propagate_batch(xt0s, Us, Ss) -> (B, n_xt) FloatingPointError listing bad intervals
  .linearize_batch(xt0s, Us, Ss) -> (ends, jx, ju, js)
  .integrate(start, param) -> IntervalResult

All arrays returned are fresh C-contiguous float64 numpy arrays; inputs are
never mutated.  The computation always runs on the GPU (``cito_*_host`` entry
points: host buffers in, H2D + kernel + D2H inside the call); device-resident
variants (`*_device`) take and return torch CUDA tensors.
"""

import sys
from dataclasses import dataclass

import numpy as np

from . import _lib
from .model import pack_model

__all__ = ["Discretizer", "AugmentedState", "IntervalParameterization", "IntervalResult", "install"]


@dataclass
class AugmentedState:
    """Same fields as cito.augmentation.AugmentedState (augmentation.py:61-76)."""

    q: np.ndarray
    v: np.ndarray
    y: np.ndarray

    def flat(self):
        return np.concatenate([np.asarray(self.q), np.asarray(self.v), np.asarray(self.y)])

    @classmethod
    def from_flat(cls, model, n_y, vec):
        vec = np.asarray(vec, dtype=float)
        n_q = 3 * len(model.links)
        return cls(q=vec[:n_q], v=vec[n_q: 2 * n_q], y=vec[2 * n_q: 2 * n_q + n_y])


@dataclass
class IntervalParameterization:
    U: np.ndarray
    S: float


@dataclass
class IntervalResult:
    end_state: AugmentedState
    jac_state: np.ndarray
    jac_U: np.ndarray
    jac_S: np.ndarray


def _ref_types():
    """Use the reference's own result types when the reference package is loaded."""
    mod = sys.modules.get("cito.augmentation")
    if mod is not None and hasattr(mod, "IntervalResult"):
        return mod.AugmentedState, mod.IntervalResult
    return AugmentedState, IntervalResult


class Discretizer:
    def __init__(self, model, mixing=None, path_fn=None, substeps=10):
        if substeps < 1:
            raise ValueError("substeps must be >= 1")
        self.model = model
        self.mixing = None if mixing is None else np.asarray(mixing, dtype=float)
        self.path_fn = path_fn
        self.substeps = substeps
        n_g_out = 0 if self.mixing is None else self.mixing.shape[0]
        n_c = len(model.contacts)
        self.n_y = 5 * n_c + n_g_out
        self.n_xt = 2 * 3 * len(model.links) + self.n_y
        self._desc = pack_model(model, self.mixing, path_fn)
        self._h = _lib.Handle(self._desc, substeps)
        d = self._h.dims
        self.n_u = d.n_u
        if d.n_xt != self.n_xt or d.n_y != self.n_y:
            raise RuntimeError(f"library dims (n_xt={d.n_xt}, n_y={d.n_y}) disagree with the model "
                               f"(n_xt={self.n_xt}, n_y={self.n_y})")

    # -- input normalisation (mirrors jnp.asarray(...).reshape(len(Ss), -1))
    def _batch(self, xt0s, Us, Ss):
        Ss = np.ascontiguousarray(np.asarray(Ss, dtype=np.float64).reshape(-1))
        B = Ss.shape[0]
        xt0s = np.ascontiguousarray(np.asarray(xt0s, dtype=np.float64).reshape(B, self.n_xt))
        Us = np.ascontiguousarray(np.asarray(Us, dtype=np.float64).reshape(B, 2 * self.n_u))
        return xt0s, Us, Ss, B

    def propagate(self, xt0, U, S):
        """End state only (augmentation.py:218-224)."""
        xt0s, Us, Ss, B = self._batch(np.asarray(xt0).reshape(1, -1), np.asarray(U).reshape(1, -1), [float(S)])
        ends = np.empty((1, self.n_xt))
        bad = np.zeros(1, dtype=np.int32)
        st = self._h.L.cito_propagate_host(self._h.ptr, 1, xt0s.ctypes.data, Us.ctypes.data, Ss.ctypes.data,
                                            ends.ctypes.data, bad.ctypes.data)
        if st == _lib.CITO_ERR_NONFINITE:
            raise FloatingPointError("non-finite state during interval integration")
        self._h.check(st, "propagate")
        return ends[0]

    def propagate_batch(self, xt0s, Us, Ss):
        """Vectorized end states (augmentation.py:226-234)."""
        xt0s, Us, Ss, B = self._batch(xt0s, Us, Ss)
        ends = np.empty((B, self.n_xt))
        bad = np.zeros(B, dtype=np.int32)
        if B == 0:
            return ends
        st = self._h.L.cito_propagate_host(self._h.ptr, B, xt0s.ctypes.data, Us.ctypes.data, Ss.ctypes.data,
                                            ends.ctypes.data, bad.ctypes.data)
        if st == _lib.CITO_ERR_NONFINITE:
            raise FloatingPointError(f"non-finite state in intervals {np.where(bad != 0)[0].tolist()}")
        self._h.check(st, "propagate_batch")
        return ends

    def linearize_batch(self, xt0s, Us, Ss, out=None):
        """End states and Jacobians (d/dstate, d/dU, d/dS) (augmentation.py:236-242).

        ``out`` (extension, not in the reference signature): caller-owned
        C-contiguous float64 arrays (ends (B, n_xt), jx (B, n_xt, n_xt),
        ju (B, n_xt, 2 n_u), js (B, n_xt)) to write into -- e.g. page-locked
        buffers reused across calls, which lets the chunked device->host
        pipeline of ``cito_linearize_host`` run fully asynchronously."""
        xt0s, Us, Ss, B = self._batch(xt0s, Us, Ss)
        n, nu2 = self.n_xt, 2 * self.n_u
        if out is None:
            ends = np.empty((B, n))
            jx = np.empty((B, n, n))
            ju = np.empty((B, n, nu2))
            js = np.empty((B, n))
        else:
            ends, jx, ju, js = out
            for a, shp in ((ends, (B, n)), (jx, (B, n, n)), (ju, (B, n, nu2)), (js, (B, n))):
                if a.shape != shp or a.dtype != np.float64 or not a.flags.c_contiguous:
                    raise ValueError(f"out array must be C-contiguous float64 of shape {shp}")
        bad = np.zeros(B, dtype=np.int32)
        if B == 0:
            return ends, jx, ju, js
        st = self._h.L.cito_linearize_host(self._h.ptr, B, xt0s.ctypes.data, Us.ctypes.data, Ss.ctypes.data,
                                            ends.ctypes.data, jx.ctypes.data, ju.ctypes.data, js.ctypes.data,
                                            bad.ctypes.data)
        if st == _lib.CITO_ERR_NONFINITE:
            # the reference raises from its propagate_batch pass (augmentation.py:238 -> :231-233)
            raise FloatingPointError(f"non-finite state in intervals {np.where(bad != 0)[0].tolist()}")
        self._h.check(st, "linearize_batch")
        return ends, jx, ju, js

    def integrate(self, start, param):
        """Single-interval integration returning an IntervalResult (augmentation.py:244-255)."""
        AS, IR = _ref_types()
        xt0 = start.flat() if hasattr(start, "flat") and callable(start.flat) else np.asarray(start)
        U_flat = np.asarray(param.U, dtype=float).reshape(-1)
        ends, jx, ju, js = self.linearize_batch(np.asarray(xt0)[None], U_flat[None], [float(param.S)])
        return IR(end_state=AS.from_flat(self.model, self.n_y, ends[0]), jac_state=jx[0], jac_U=ju[0],
                  jac_S=js[0])

    # -- device-resident variants (torch CUDA tensors, caller's current stream)
    def linearize_batch_device(self, xt0s, Us, Ss, out=None, stream=None):
        import torch

        B = Ss.shape[0]
        n, nu2 = self.n_xt, 2 * self.n_u
        dev = xt0s.device
        if out is None:
            out = (torch.empty((B, n), dtype=torch.float64, device=dev),
                   torch.empty((B, n, n), dtype=torch.float64, device=dev),
                   torch.empty((B, n, nu2), dtype=torch.float64, device=dev),
                   torch.empty((B, n), dtype=torch.float64, device=dev),
                   torch.empty((B,), dtype=torch.int32, device=dev))
        ends, jx, ju, js, bad = out
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        self._h.check(self._h.L.cito_linearize_dev(self._h.ptr, B, xt0s.data_ptr(), Us.data_ptr(), Ss.data_ptr(),
                                                 ends.data_ptr(), jx.data_ptr(), ju.data_ptr(), js.data_ptr(),
                                                 bad.data_ptr(), s), "linearize_dev")
        return out

    def propagate_batch_device(self, xt0s, Us, Ss, out=None, stream=None):
        import torch

        B = Ss.shape[0]
        dev = xt0s.device
        if out is None:
            out = (torch.empty((B, self.n_xt), dtype=torch.float64, device=dev),
                   torch.empty((B,), dtype=torch.int32, device=dev))
        ends, bad = out
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        self._h.check(self._h.L.cito_propagate_dev(self._h.ptr, B, xt0s.data_ptr(), Us.data_ptr(), Ss.data_ptr(),
                                                 ends.data_ptr(), bad.data_ptr(), s), "propagate_dev")
        return out

    def launch_count(self):
        return self._h.launch_count()


def install(tr):
    """Swap a reference ``cito.ocp.Transcription``'s discretizer for the GPU one
    (the reference holds it as ``tr.discretizer``, ocp.py:263-265)."""
    tr.discretizer = Discretizer(tr.model, mixing=tr.mixing, path_fn=tr.path_fn,
                                 substeps=tr.scenario.substeps)
    return tr.discretizer
