"""Multi-GPU plumbing for the GP loop (one process per GPU, torch.distributed):
the launcher environment, the object slabs of the sharded loop (shard.py,
partition.py), the replica seeds of ``bench.py --mode replicas`` and the
max-over-ranks timing reduction of ``bench.py``.  Because rho is int64 fixed
point (2^-40 per unit density), the all-reduced density map of the sharded
loop is bit-identical to the single-GPU map for any number of ranks and any
reduction order — the property ``tests/test_dist.py`` checks with the gloo
backend on CPU.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def rank_world():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard_range(n, rank, world):
    """Contiguous slab [lo, hi) of n units owned by `rank` (sizes differ by <= 1)."""
    q, r = divmod(int(n), int(world))
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def object_slabs(n_inst, n_fill, rank, world):
    """This rank's objects in the sharded loop: (instance slab size padded to
    equal slabs, (i0, i1) instance range, (f0, f1) filler range in object
    indices).  Equal padded instance slabs make the owner-sum reduce-scatter
    and the position all-gather equal-count collectives."""
    slab = -(-n_inst // world) if n_inst else 0
    inst = (min(rank * slab, n_inst), min((rank + 1) * slab, n_inst))
    lo, hi = shard_range(n_fill, rank, world)
    return slab, inst, (n_inst + lo, n_inst + hi)


def replica_seed(base_seed, rank):
    """Seed of the independent placement a rank runs in replica mode."""
    return int(base_seed) + int(rank)


def max_over_ranks(values):
    """Element-wise max of a list of floats over all ranks (timings)."""
    t = torch.tensor(list(values), dtype=torch.float64,
                     device="cuda" if dist.is_initialized() and
                     dist.get_backend() == "nccl" else "cpu")
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]
