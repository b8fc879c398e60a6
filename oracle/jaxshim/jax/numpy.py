"""``jax.numpy`` subset on torch float64 (TEST INFRASTRUCTURE ONLY; see __init__)."""

import numpy as _np
import torch

ndarray = torch.Tensor
float64 = torch.float64
pi = _np.pi


def _dt(dtype):
    if dtype is None or dtype is float or dtype is _np.float64 or dtype == "float64":
        return torch.float64
    if dtype is int:
        return torch.int64
    return dtype


def _has_tensor(obj):
    if isinstance(obj, torch.Tensor):
        return True
    if isinstance(obj, (list, tuple)):
        return any(_has_tensor(o) for o in obj)
    return False


def _build(obj):
    if isinstance(obj, torch.Tensor):
        return obj.to(torch.float64) if obj.is_floating_point() else obj.to(torch.float64)
    if isinstance(obj, (list, tuple)):
        return torch.stack([_build(o) for o in obj])
    return torch.tensor(float(obj), dtype=torch.float64)


def asarray(a, dtype=None):
    if isinstance(a, torch.Tensor):
        if dtype is not None and _dt(dtype) != a.dtype:
            return a.to(_dt(dtype))
        return a
    if _has_tensor(a):
        return _build(a)
    arr = _np.asarray(a)
    if dtype is None and arr.dtype.kind in "biu":
        return torch.as_tensor(arr)
    return torch.as_tensor(arr.astype(_np.float64))


def array(a, dtype=None):
    if _has_tensor(a):
        return _build(a)
    return asarray(_np.array(a, dtype=_np.float64 if dtype in (None, float) else dtype))


def zeros(shape, dtype=None):
    return torch.zeros(shape, dtype=_dt(dtype))


def ones(shape, dtype=None):
    return torch.ones(shape, dtype=_dt(dtype))


def arange(*a):
    return torch.arange(*a, dtype=torch.float64)


def concatenate(xs, axis=0):
    return torch.cat([asarray(x) for x in xs], dim=axis)


def stack(xs, axis=0):
    return torch.stack([asarray(x) for x in xs], dim=axis)


def atleast_1d(x):
    return torch.atleast_1d(asarray(x))


def diag(x):
    return torch.diag(asarray(x))


def dot(a, b):
    a, b = asarray(a), asarray(b)
    if a.dim() == 1 and b.dim() == 1:
        return torch.dot(a, b)
    return a @ b


def sqrt(x):
    return torch.sqrt(asarray(x))


def sin(x):
    return torch.sin(asarray(x))


def cos(x):
    return torch.cos(asarray(x))


def abs(x):  # noqa: A001
    return torch.abs(asarray(x))


def where(c, a, b):
    return torch.where(asarray(c), asarray(a), asarray(b))


def maximum(a, b):
    return torch.maximum(asarray(a), asarray(b))


def minimum(a, b):
    return torch.minimum(asarray(a), asarray(b))


def exp(x):
    return torch.exp(asarray(x))


def log(x):
    return torch.log(asarray(x))


def power(a, b):
    return torch.pow(asarray(a), b if isinstance(b, (int, float)) else asarray(b))


class linalg:  # noqa: N801
    @staticmethod
    def solve(a, b):
        return torch.linalg.solve(asarray(a), asarray(b))

    @staticmethod
    def norm(a):
        return torch.linalg.norm(asarray(a))
