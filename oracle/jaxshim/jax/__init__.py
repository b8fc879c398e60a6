"""Minimal ``jax`` stand-in backed by ``torch.func`` (TEST INFRASTRUCTURE ONLY).

JAX is not installed in this image and cannot be (no network).  This shim
lets the *unmodified* reference package ``cito`` (``/root/reference/pkg/src``)
import and run on CPU so that it can produce golden vectors for the parity
tests.  It is never imported by the product path (``paper_2604_09993_b200``);
only ``oracle/ref_runner.py`` (and through it ``tests/golden/make_golden.py``)
puts it on ``sys.path``.

Mapping (what the reference uses):
  jit -> identity; vmap -> per-element Python loop (torch.func.vmap over the
  nested jacfwd+solve returned NaN for batch elements >= 1); jacfwd/jvp/grad
  -> torch.func; lax.scan -> loop; jnp.* -> torch float64; ``x.at[i].add``
  -> out-of-place one-hot add; jax.core.Tracer -> torch.Tensor.
"""

import types

import numpy as _np
import torch

torch.set_default_dtype(torch.float64)

from . import numpy  # noqa: E402,F401  (jax.numpy)
from . import lax  # noqa: E402,F401
from . import core  # noqa: E402,F401


class _Config:
    def update(self, key, value):
        return None


config = _Config()


def _to_t(a):
    if isinstance(a, torch.Tensor):
        return a
    return torch.as_tensor(_np.asarray(a, dtype=_np.float64))


def jit(f=None, **kw):
    if f is None:
        return lambda g: g
    return f


def _tuplify(x):
    return x if isinstance(x, tuple) else (x,)


def jacfwd(f, argnums=0):
    def wrapped(*args):
        args = tuple(_to_t(a) for a in args)
        return torch.func.jacfwd(f, argnums=argnums)(*args)

    return wrapped


def grad(f, argnums=0):
    def wrapped(*args):
        args = tuple(_to_t(a) for a in args)
        return torch.func.grad(f, argnums=argnums)(*args)

    return wrapped


def jvp(f, primals, tangents):
    primals = tuple(_to_t(p) for p in primals)
    tangents = tuple(_to_t(t) for t in tangents)
    return torch.func.jvp(f, primals, tangents)


def vmap(f, in_axes=0):
    """Loop-based vmap over axis 0 (only in_axes 0 / None are used)."""

    def wrapped(*args):
        axes = in_axes if isinstance(in_axes, (tuple, list)) else (in_axes,) * len(args)
        n = None
        for a, ax in zip(args, axes):
            if ax is not None:
                n = len(a)
                break
        outs = []
        for i in range(n):
            call = [(_to_t(a)[i] if ax is not None else a) for a, ax in zip(args, axes)]
            outs.append(f(*call))
        if isinstance(outs[0], tuple):
            return tuple(torch.stack([o[j] for o in outs]) for j in range(len(outs[0])))
        return torch.stack(outs)

    return wrapped


# ``x.at[i].add(v)`` functional update used by multibody.generalized_forces
class _AtIndexer:
    def __init__(self, t):
        self._t = t

    def __getitem__(self, idx):
        t = self._t

        class _Upd:
            def add(self_inner, v):
                onehot = torch.zeros(t.shape, dtype=t.dtype)
                onehot[idx] = 1.0
                return t + onehot * v

            def set(self_inner, v):
                onehot = torch.zeros(t.shape, dtype=t.dtype)
                onehot[idx] = 1.0
                return t * (1.0 - onehot) + onehot * v

        return _Upd()


if not hasattr(torch.Tensor, "at"):
    torch.Tensor.at = property(lambda self: _AtIndexer(self))

__all__ = ["jit", "vmap", "jacfwd", "jvp", "grad", "config", "numpy", "lax", "core"]
