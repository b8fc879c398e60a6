"""Multi-GPU sharding of independent linearization work.

Multiple shooting makes every interval (and every multi-start problem)
independent (the reference's own thread fan-out relies on it and
returns results identical to the serial path, cito/scp.py:101-112), so there is
no exchange inside the computation.  One process per GPU (torch.distributed,
NCCL over NVLink): each rank linearizes a contiguous shard on its own device and
the results are collected on rank 0 once, for result collection only:

  ShardedBatch       configs[2]: a batch of B independent intervals, contiguous
                     interval ranges per rank (4096 -> 512 per GPU at 8 GPUs)
  ShardedMultiStart  configs[3]: P multi-start problems (initial guesses with
                     seeds), whole problems per rank (1024 -> 128 per GPU), so
                     a problem's intervals and node relations stay on one GPU

Collection (``collect=``):
  "device"  one grouped NCCL send/recv (torch batch_isend_irecv -> ncclGroup of
            ncclSend/ncclRecv): every rank's output slices land directly in the
            matching rows of rank 0's full device arrays (no staging, no copy
            afterwards); rank 0's own shard is computed in place
  "host"    the N-parallel-D2H alternative: rank 0 creates one shared-memory host
            buffer, every rank registers it (page-locked) and copies its rows
            straight into it; rank 0 returns numpy views of the full result
  "none"    each rank keeps its shard (returned as device tensors)

Row order of a collected result equals the single-GPU call on the whole batch,
and the bits are the same as long as every shard runs the same kernel
generation as the whole batch (the K1 dispatch depends on the batch size,
capi `launch_linearize`); tests/test_multigpu.py checks bit-equality.

  shard_range(n, rank, world)   contiguous [lo, hi) split, remainder spread over low ranks
  gather_rows(x, group=None)    all_gather of a (rows, ...) tensor with per-rank row counts
"""

import numpy as np

__all__ = ["shard_range", "shard_bounds", "gather_rows", "gather_slices", "HostResult", "ShardedBatch",
           "ShardedMultiStart", "multistart_intervals", "problem_metrics"]


def shard_range(n, rank, world):
    """Contiguous shard of n items for `rank` of `world` (sizes differ by at most 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_bounds(n, world):
    return [shard_range(n, r, world) for r in range(world)]


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return None
    return dist


def _world(group):
    dist = _dist()
    if dist is None:
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _global_rank(group, r):
    import torch.distributed as dist

    return r if group is None else dist.get_global_rank(group, r)


def gather_slices(local, full, rows_per_unit, bounds, group=None):
    """Collect per-rank row slices into rank 0's full arrays with one grouped
    send/recv (NCCL: one ncclGroupStart/End with a ncclSend per array on every
    rank > 0 and the matching ncclRecv's on rank 0).

    local:  {name: tensor} this rank's rows (contiguous, first dim = units * rows_per_unit[name])
    full:   {name: tensor} on rank 0 the full arrays (rank 0's own rows already in place), else None
    bounds: [(lo, hi)] unit ranges of every rank; rows_per_unit[name] rows per unit.
    With the gloo backend (CPU tests) device tensors are staged through host memory."""
    import torch
    import torch.distributed as dist

    rank, world = _world(group)
    if world == 1:
        return full
    staged = dist.get_backend(group) == "gloo"
    ops, post = [], []
    names = sorted(local)
    if rank == 0:
        for r in range(1, world):
            lo, hi = bounds[r]
            if hi <= lo:
                continue
            for k in names:
                dst = full[k][lo * rows_per_unit[k]: hi * rows_per_unit[k]]
                buf = torch.empty(dst.shape, dtype=dst.dtype) if staged and dst.is_cuda else dst
                ops.append(dist.P2POp(dist.irecv, buf, _global_rank(group, r), group))
                if buf is not dst:
                    post.append((dst, buf))
    else:
        lo, hi = bounds[rank]
        if hi > lo:
            for k in names:
                src = local[k]
                if staged and src.is_cuda:
                    src = src.cpu()
                ops.append(dist.P2POp(dist.isend, src, _global_rank(group, 0), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for dst, buf in post:
        dst.copy_(buf)
    return full


class HostResult:
    """Full result arrays on the host, written by every rank into one shared-memory
    buffer (the N-parallel-D2H collection).  Rank 0 owns the segment; the arrays
    (numpy views) stay valid while this object lives."""

    def __init__(self, shapes, group=None):
        import torch
        import torch.distributed as dist
        from multiprocessing import shared_memory

        self.rank, world = _world(group)
        self.layout, off = {}, 0
        for k, (shape, dtype) in sorted(shapes.items()):
            n = int(np.prod(shape)) * np.dtype(dtype).itemsize
            off = (off + 255) // 256 * 256
            self.layout[k] = (off, shape, dtype)
            off += n
        self.nbytes = max(256, (off + 4095) // 4096 * 4096)
        name = [None]
        if self.rank == 0:
            self.shm = shared_memory.SharedMemory(create=True, size=self.nbytes)
            name[0] = self.shm.name
        if world > 1:
            dist.broadcast_object_list(name, src=_global_rank(group, 0), group=group)
        if self.rank != 0:
            self.shm = shared_memory.SharedMemory(name=name[0])
            try:  # the segment belongs to rank 0: keep this process's tracker from unlinking it at exit
                from multiprocessing import resource_tracker

                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.buf = np.ndarray((self.nbytes,), dtype=np.uint8, buffer=self.shm.buf)
        self.arrays = {k: self.buf[o: o + int(np.prod(s)) * np.dtype(d).itemsize].view(d).reshape(s)
                       for k, (o, s, d) in self.layout.items()}
        self.tensors = {k: torch.from_numpy(v) for k, v in self.arrays.items()}
        cudart = torch.cuda.cudart()
        # page-lock the shared segment so the D2H copies are true async DMA (cudaHostRegisterPortable)
        self._registered = int(cudart.cudaHostRegister(self.buf.ctypes.data, self.nbytes, 1)) == 0

    def close(self):
        import torch

        if getattr(self, "_registered", False):
            torch.cuda.cudart().cudaHostUnregister(self.buf.ctypes.data)
            self._registered = False
        self.arrays, self.tensors, self.buf = {}, {}, None
        try:
            self.shm.close()
            if self.rank == 0:
                self.shm.unlink()
        except (FileNotFoundError, BufferError):
            pass

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _host_collect(local, host, rows_per_unit, lo, group):
    """Every rank copies its rows into the shared host result (async on the current
    stream), then synchronizes and meets the others at a barrier."""
    import torch
    import torch.distributed as dist

    for k, v in local.items():
        dst = host.tensors[k][lo * rows_per_unit[k]: lo * rows_per_unit[k] + v.shape[0]]
        dst.copy_(v, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    if _dist() is not None:
        dist.barrier(group=group)


class ShardedBatch:
    """configs[2]: ``Discretizer.linearize_batch`` (augmentation.py:236-242) of one
    batch of independent intervals spread over the ranks of ``group``.

    Every rank passes the same full batch (host arrays or tensors); only its own
    rows are copied to its GPU."""

    FIELDS = ("ends", "jx", "ju", "js", "bad")

    def __init__(self, disc, group=None, device=None):
        import torch

        self.disc, self.group = disc, group
        self.rank, self.world = _world(group)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self._buf = {}

    def bounds(self, B):
        return shard_bounds(B, self.world)

    def _alloc(self, B):
        import torch

        n, nu2 = self.disc.n_xt, 2 * self.disc.n_u
        f = dict(dtype=torch.float64, device=self.device)
        return {"ends": torch.empty((B, n), **f), "jx": torch.empty((B, n, n), **f),
                "ju": torch.empty((B, n, nu2), **f), "js": torch.empty((B, n), **f),
                "bad": torch.empty((B,), dtype=torch.int32, device=self.device)}

    def shapes(self, B):
        n, nu2 = self.disc.n_xt, 2 * self.disc.n_u
        return {"ends": ((B, n), np.float64), "jx": ((B, n, n), np.float64), "ju": ((B, n, nu2), np.float64),
                "js": ((B, n), np.float64), "bad": ((B,), np.int32)}

    def compute(self, xt0s, Us, Ss):
        """Linearize this rank's shard on its GPU.  Inputs: the full batch (host
        arrays, or tensors -- only rows [lo, hi) are read).  Returns ({name: device
        tensor} of the shard -- on rank 0 a view into the full-batch buffers --,
        (lo, hi), B)."""
        import torch

        B = int(Ss.shape[0]) if torch.is_tensor(Ss) else int(np.asarray(Ss).reshape(-1).shape[0])
        lo, hi = shard_range(B, self.rank, self.world)
        if self.rank == 0:
            key = ("full", B)
            if key not in self._buf:
                self._buf[key] = self._alloc(B)
            out = {k: v[lo:hi] for k, v in self._buf[key].items()}
        else:
            key = ("part", hi - lo)
            if key not in self._buf:
                self._buf[key] = self._alloc(hi - lo)
            out = self._buf[key]
        if hi > lo:
            dev = self.device

            def part(a, cols):
                if torch.is_tensor(a):
                    return a.reshape(B, cols)[lo:hi].to(dev).contiguous()
                return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(B, cols)[lo:hi]),
                                       device=dev)

            self.disc.linearize_batch_device(part(xt0s, self.disc.n_xt), part(Us, 2 * self.disc.n_u),
                                             part(Ss, 1).reshape(-1), out=tuple(out[k] for k in self.FIELDS))
        return out, (lo, hi), B

    def linearize(self, xt0s, Us, Ss, collect="device", host=None):
        """Shard, compute, collect.  Returns on rank 0: collect="device" -> dict of
        full device tensors; "host" -> dict of numpy arrays (shared-memory views;
        ``host`` = a reusable HostResult of ``shapes(B)``); "none" -> this rank's
        shard on every rank.  Other ranks return None for "device"/"host"."""
        out, (lo, hi), B = self.compute(xt0s, Us, Ss)
        return self._collect(out, B, lo, collect, host)

    def _collect(self, out, B, lo, collect, host):
        import torch

        rows = {k: 1 for k in self.FIELDS}
        if collect == "none":
            return out
        if collect == "device":
            full = self._buf.get(("full", B)) if self.rank == 0 else None
            gather_slices(out, full, rows, self.bounds(B), self.group)
            if self.rank == 0:
                torch.cuda.current_stream(self.device).synchronize()
                if bool((full["bad"] != 0).any()):
                    bad = torch.nonzero(full["bad"]).flatten().tolist()
                    raise FloatingPointError(f"non-finite state in intervals {bad}")
                return full
            return None
        if collect == "host":
            h = host if host is not None else HostResult(self.shapes(B), self.group)
            _host_collect(out, h, rows, lo, self.group)
            if self.rank == 0:
                if h.arrays["bad"].any():
                    raise FloatingPointError(f"non-finite state in intervals {np.where(h.arrays['bad'])[0].tolist()}")
                return h.arrays if host is not None else dict(h.arrays, _owner=h)
            return None
        raise ValueError(f"collect must be 'device', 'host' or 'none', not {collect!r}")


class ShardedMultiStart:
    """configs[3]: ``linearize_all`` (scp.py:87-135) of P multi-start problems -- the
    scenario's ``initial_guess`` (ocp.py:461-505) for each seed -- with whole problems
    per rank.  ``seeds`` is the global list; each rank builds and linearizes only its
    own problems (batched initial guess, one K1 + one K3 launch per call)."""

    def __init__(self, scenario, seeds, group=None, device=None):
        import torch

        from .linearize import GpuTranscription, initial_guess_batch

        self.group = group
        self.rank, self.world = _world(group)
        if device is not None and not isinstance(device, int):
            device = torch.device(device).index
        self.gt = GpuTranscription(scenario, device=device)
        self.device = self.gt.device
        self.P = len(seeds)
        self.all_bounds = shard_bounds(self.P, self.world)
        self.lo, self.hi = self.all_bounds[self.rank]
        my = list(seeds)[self.lo: self.hi]
        self.Z = initial_guess_batch(scenario, self.gt.disc, my, self.gt.lay) if my else np.zeros((0, self.gt.lay.dim))
        self.Z_dev = torch.as_tensor(self.Z, device=self.device)
        lay = self.gt.lay
        self.rows = {k: (lay.N - 1 if v.shape[0] == 1 * (lay.N - 1) else lay.N)
                     for k, v in self.gt._alloc_out(1).items()}
        self.full = self.gt._alloc_out(self.P) if self.rank == 0 else None
        if self.rank == 0:
            self.out = {k: v[self.lo * self.rows[k]: self.hi * self.rows[k]] for k, v in self.full.items()}
        else:
            self.out = self.gt._alloc_out(max(0, self.hi - self.lo))

    def shapes(self):
        import torch

        return {k: ((self.P * self.rows[k],) + tuple(v.shape[1:]), np.int32 if v.dtype == torch.int32 else np.float64)
                for k, v in self.out.items()}

    def compute(self, delta, epsilon=None):
        if self.hi > self.lo:
            self.gt.linearize_device(self.Z_dev, delta, epsilon, out=self.out)
        return self.out

    def linearize(self, delta, epsilon=None, collect="device", host=None):
        import torch

        self.compute(delta, epsilon)
        if collect == "none":
            return self.out
        if collect == "device":
            gather_slices(self.out, self.full, self.rows, self.all_bounds, self.group)
            if self.rank == 0:
                torch.cuda.current_stream(self.device).synchronize()
                if bool((self.full["bad"] != 0).any()):
                    raise FloatingPointError("non-finite state in intervals "
                                             f"{torch.nonzero(self.full['bad']).flatten().tolist()}")
                return self.full
            return None
        if collect == "host":
            h = host if host is not None else HostResult(self.shapes(), self.group)
            _host_collect(self.out, h, self.rows, self.lo, self.group)
            if self.rank == 0:
                return h.arrays if host is not None else dict(h.arrays, _owner=h)
            return None
        raise ValueError(f"collect must be 'device', 'host' or 'none', not {collect!r}")


def multistart_intervals(sc, seeds, disc):
    """Stack the N-1 intervals of the initial guesses for each seed (cito/ocp.py:461-505)."""
    from .linearize import initial_guess_batch
    from .scenario import Layout

    lay = Layout(sc)
    Z = initial_guess_batch(sc, disc, list(seeds), lay)
    n = lay.N - 1
    xs = np.concatenate([np.stack([z[lay.xp(k)] for k in range(n)]) for z in Z])
    us = np.concatenate([np.stack([z[lay.u(k)] for k in range(n)]) for z in Z])
    ss = np.concatenate([np.array([z[lay.s(k)][0] for k in range(n)]) for z in Z])
    return xs, us, ss, Z, lay


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
