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
