"""``jax.lax.scan`` as a Python loop (TEST INFRASTRUCTURE ONLY; see __init__)."""

import torch


def scan(f, init, xs):
    carry = init
    ys = []
    for i in range(len(xs)):
        carry, y = f(carry, xs[i])
        ys.append(y)
    if ys and ys[0] is not None:
        ys = torch.stack(ys)
    else:
        ys = None
    return carry, ys
