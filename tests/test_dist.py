"""Host-side multi-process logic with the gloo backend (world_size 2, CPU).

* slab partitioning covers every unit exactly once;
* per-rank fixed-point density maps of disjoint object slabs, all-reduced,
  equal the single-process map bit for bit (the property that makes the
  config-4 sharded path exact for any GPU count);
* the max-over-ranks timing reduction used by bench.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_09070_b200.dist import max_over_ranks, replica_seed, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import fixed as FX
        from oracle import port as P

        rng = np.random.default_rng(3)
        grid = P.Grid(40.0, 30.0, 16, 12, 2)
        n = 500
        w = rng.uniform(0.5, 4, n)
        h = rng.uniform(0.5, 4, n)
        cl = P.Cloud(rng.uniform(0, 40, n), rng.uniform(0, 30, n),
                     rng.uniform(grid.dz / 4, 3 * grid.dz / 4, n), w, h,
                     np.full(n, grid.dz / 2), np.ones(n), rng.random(n) < 0.05)
        lo, hi = shard_range(n, rank, world)
        part = torch.from_numpy(FX.fixed_rho(grid, cl.take(np.arange(lo, hi))).reshape(-1).copy())
        dist.all_reduce(part)  # int64: the sum is exact in any order
        full = FX.fixed_rho(grid, cl).reshape(-1)
        ok = bool(np.array_equal(part.numpy(), full))
        mx = max_over_ranks([1.0 + rank, 5.0 - rank])
        out[rank] = (ok, mx)
    finally:
        dist.destroy_process_group()


def test_shard_range_covers():
    for n in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1
    assert replica_seed(1, 3) == 4


def test_gloo_world2_fixed_point_allreduce_exact():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert all(res[r][0] for r in range(world))
    assert all(res[r][1] == [2.0, 5.0] for r in range(world))


def test_object_slabs_cover_every_object_once():
    from paper_2403_09070_b200.dist import object_slabs

    for I, F in ((0, 0), (1, 0), (10, 3), (1001, 77), (800064, 40000)):
        for world in (1, 2, 3, 8):
            seen = np.zeros(I + F, dtype=int)
            slab = None
            for r in range(world):
                s, (i0, i1), (f0, f1) = object_slabs(I, F, r, world)
                slab = s if slab is None else slab
                assert s == slab and i1 - i0 <= s and i0 == min(r * s, I)
                seen[i0:i1] += 1
                seen[f0:f1] += 1
                assert I <= f0 <= f1 <= I + F
            assert np.all(seen == 1)


def _comm_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_09070_b200.shard import ShardComm

        c = ShardComm()
        n = 5
        buf = torch.arange(world * n, dtype=torch.float64) + 100 * rank
        c.reduce_scatter_chunks(buf, n)  # own chunk = sum over ranks of that chunk
        mine = buf[rank * n:(rank + 1) * n].clone()
        g = torch.zeros(world * n, dtype=torch.float64)
        g[rank * n:(rank + 1) * n] = rank + 1
        c.all_gather_chunks(g, n)
        t = torch.tensor([float(rank)])
        c.all_reduce(t, dist.ReduceOp.MAX)
        out[rank] = (mine.tolist(), g.tolist(), float(t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_collectives():
    """The sharded loop's collectives (shard.ShardComm) on CPU tensors with gloo:
    reduce-scatter of equal slabs, all-gather of slabs, max all-reduce."""
    world, n = 2, 5
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_comm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        mine, g, t = res[r]
        base = np.arange(world * n, dtype=float)[r * n:(r + 1) * n]
        assert mine == list(world * base + 100 * sum(range(world)))
        assert g == [float(k // n + 1) for k in range(world * n)]
        assert t == world - 1
