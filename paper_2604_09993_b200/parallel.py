"""Multi-GPU sharding of independent linearization work.

Multiple shooting makes every interval (and every multi-start problem)
independent (the reference's own thread fan-out relies on it,
cito/scp.py:101-112), so there is no exchange inside the computation: each
rank (one process per GPU, torch.distributed over NCCL) linearizes a
contiguous shard, and a single collective collects per-problem results.

  shard_range(n, rank, world)        contiguous [lo, hi) split, remainder spread over low ranks
  multistart_intervals(sc, seeds, disc)  interval batch of several initial guesses (configs[3])
  gather_rows(x, group=None)         all_gather of a (rows, ...) tensor with per-rank row counts
"""

import numpy as np

__all__ = ["shard_range", "multistart_intervals", "gather_rows", "problem_metrics"]


def shard_range(n, rank, world):
    """Contiguous shard of n items for `rank` of `world` (sizes differ by at most 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def multistart_intervals(sc, seeds, disc):
    """Stack the N-1 intervals of the initial guesses for each seed (cito/ocp.py:461-505)."""
    from .linearize import initial_guess
    from .scenario import Layout

    lay = Layout(sc)
    xs, us, ss, zs = [], [], [], []
    for seed in seeds:
        z = initial_guess(sc, disc, lay, seed=int(seed))
        zs.append(z)
        xs.append(np.stack([z[lay.xp(k)] for k in range(lay.N - 1)]))
        us.append(np.stack([z[lay.u(k)] for k in range(lay.N - 1)]))
        ss.append(np.array([z[lay.s(k)][0] for k in range(lay.N - 1)]))
    return np.concatenate(xs), np.concatenate(us), np.concatenate(ss), np.stack(zs), lay


def problem_metrics(ends, zs_next_xm, n_int):
    """Per-problem max |defect| (the multiple-shooting residual, cito/scp.py:115),
    from interval ends (P*n_int, n_xt) and the matching z[xm(k+1)] rows."""
    d = (zs_next_xm - ends).reshape(-1, n_int, ends.shape[-1])
    return d.abs().amax(dim=(1, 2)) if hasattr(d, "abs") else np.abs(d).max(axis=(1, 2))


def gather_rows(x, group=None):
    """all_gather along dim 0 with possibly different row counts per rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([x.shape[0]], dtype=torch.int64, device=x.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    m = max(ns)
    pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:k] for o, k in zip(outs, ns)])
