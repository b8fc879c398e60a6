"""N>1 path on CPU: world_size-2 gloo process group exercising the sharding and
the result-collection collective of paper_2604_09993_b200.parallel, with the
CPU oracle standing in for the per-rank GPU work (checker only)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_09993_b200.parallel import gather_rows, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 29, 4096, 50176):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import pyoracle
    from conftest import golden_scenario, scenario_desc

    from paper_2604_09993_b200 import synth

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc = golden_scenario("monoped_n20")
    x, U, S = synth.random_intervals(sc, 37, seed=3)
    lo, hi = shard_range(len(S), rank, world)
    ends, bad = pyoracle.propagate(scenario_desc(sc), sc.substeps, x[lo:hi], U[lo:hi], S[lo:hi])
    got = gather_rows(torch.as_tensor(ends))
    if rank == 0:
        np.save(result_path, got.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shard_and_gather(tmp_path):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import pyoracle
    from conftest import golden_scenario, scenario_desc

    from paper_2604_09993_b200 import synth

    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    sc = golden_scenario("monoped_n20")
    x, U, S = synth.random_intervals(sc, 37, seed=3)
    ref, _ = pyoracle.propagate(scenario_desc(sc), sc.substeps, x, U, S)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)  # same per-interval arithmetic, order restored by the gather


def _gather_worker(rank, world, port, result_path):
    """gather_slices with gloo on CPU tensors: uneven shards of two arrays with
    different rows per unit land in rank 0's full arrays in order."""
    from paper_2604_09993_b200.parallel import gather_slices, shard_bounds

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    P = 7
    bounds = shard_bounds(P, world)
    lo, hi = bounds[rank]
    rows = {"a": 3, "b": 4}
    full_a = torch.arange(P * 3 * 2, dtype=torch.float64).reshape(P * 3, 2)
    full_b = -torch.arange(P * 4, dtype=torch.float64).reshape(P * 4, 1)
    local = {"a": full_a[lo * 3: hi * 3].clone(), "b": full_b[lo * 4: hi * 4].clone()}
    full = None
    if rank == 0:
        full = {"a": torch.zeros_like(full_a), "b": torch.zeros_like(full_b)}
        full["a"][lo * 3: hi * 3] = local["a"]
        full["b"][lo * 4: hi * 4] = local["b"]
    gather_slices(local, full, rows, bounds)
    if rank == 0:
        np.save(result_path, np.concatenate([full["a"].numpy().ravel(), full["b"].numpy().ravel()]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_slices_gloo(tmp_path, world):
    out = str(tmp_path / "g.npy")
    mp.spawn(_gather_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    P = 7
    ref = np.concatenate([np.arange(P * 6, dtype=float), -np.arange(P * 4, dtype=float)])
    assert np.array_equal(np.load(out), ref)


def _gpu_worker(rank, world, port, result_dir, kind):
    """Two ranks on cuda:0 over gloo (the plumbing of the NCCL path; no kernel waits on
    another rank): shard, compute on the GPU, collect on rank 0 -- device and host."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    from conftest import golden_scenario

    from paper_2604_09993_b200 import Discretizer, synth
    from paper_2604_09993_b200.parallel import HostResult, ShardedBatch, ShardedMultiStart

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc = golden_scenario("halfcheetah_n30")
    if kind == "batch":
        g, n_g = sc.path_constraints()
        disc = Discretizer(sc.model, mixing=sc.mixing_matrix(n_g), path_fn=g, substeps=sc.substeps)
        B = 2400  # every shard (1200) and the whole batch run the 3-interval lockstep kernel
        x, U, S = synth.random_intervals(sc, B, seed=11)
        sb = ShardedBatch(disc)
        full = sb.linearize(x, U, S, collect="device")
        host = HostResult(sb.shapes(B))
        hres = sb.linearize(x, U, S, collect="host", host=host)
        if rank == 0:
            for k in ("ends", "jx", "ju", "js"):
                np.save(os.path.join(result_dir, f"dev_{k}.npy"), full[k].cpu().numpy())
                np.save(os.path.join(result_dir, f"host_{k}.npy"), hres[k])
        dist.barrier()
        host.close()
    else:
        seeds = list(range(18))  # 9 x 29 intervals per rank and 18 x 29 in one launch: same K1 generation
        ms = ShardedMultiStart(sc, seeds)
        full = ms.linearize(1.0, collect="device")
        if rank == 0:
            for k, v in full.items():
                np.save(os.path.join(result_dir, f"ms_{k}.npy"), v.cpu().numpy())
            np.save(os.path.join(result_dir, "ms_Z0.npy"), ms.Z)
        dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_batch_two_ranks_equals_single_gpu(tmp_path):
    from conftest import golden_scenario

    from paper_2604_09993_b200 import Discretizer, synth

    mp.spawn(_gpu_worker, args=(2, _free_port(), str(tmp_path), "batch"), nprocs=2, join=True)
    sc = golden_scenario("halfcheetah_n30")
    g, n_g = sc.path_constraints()
    disc = Discretizer(sc.model, mixing=sc.mixing_matrix(n_g), path_fn=g, substeps=sc.substeps)
    x, U, S = synth.random_intervals(sc, 2400, seed=11)
    ref = disc.linearize_batch(x, U, S)
    for k, r in zip(("ends", "jx", "ju", "js"), ref):
        assert np.array_equal(np.load(tmp_path / f"dev_{k}.npy"), r), k
        assert np.array_equal(np.load(tmp_path / f"host_{k}.npy"), r), k


@pytest.mark.gpu
def test_sharded_multistart_two_ranks_equals_single_gpu(tmp_path):
    from conftest import golden_scenario

    from paper_2604_09993_b200.linearize import GpuTranscription, initial_guess_batch

    mp.spawn(_gpu_worker, args=(2, _free_port(), str(tmp_path), "multistart"), nprocs=2, join=True)
    sc = golden_scenario("halfcheetah_n30")
    gt = GpuTranscription(sc)
    Z = initial_guess_batch(sc, gt.disc, list(range(18)), gt.lay)
    assert np.array_equal(np.load(tmp_path / "ms_Z0.npy"), Z[:9])
    r = gt.linearize_device(torch.as_tensor(Z, device=gt.device), 1.0)
    torch.cuda.synchronize()
    for k, v in r.items():
        assert np.array_equal(np.load(tmp_path / f"ms_{k}.npy"), v.cpu().numpy()), k
