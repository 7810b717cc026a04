"""Partition of one placement over the ranks of the sharded loop.

Two host-side steps, both on the netlist alone (they run once per run):

* ``locality_order``: an instance numbering in which connected instances sit
  next to each other, by label propagation over the netlist's clique
  expansion (each pin pair of a net weighted 1 / (degree - 1), the usual
  net model): every instance repeatedly adopts the label with the largest
  total weight among its net neighbours, so the netlist's clusters (the
  ~40-instance clusters of the synthetic generator, synth.py:145-157; the
  modules of a real design) collapse onto single labels, and sorting by label
  makes them contiguous.  Contiguous instance slabs then hold whole clusters,
  and only the nets that genuinely span clusters cross ranks.
* ``HaloPlan``: with instance slabs fixed, each rank evaluates every net
  that touches its slab (a net spanning k ranks is evaluated on each of them,
  each keeping the gradients of its own pins), so the per-instance WL sums
  need no exchange at all; the net's value, exact WL and crossing flag are
  counted by its primary rank only (the owner of its first pin).  What each
  rank then needs from the others is the positions of the remote instances
  of its nets (its halo): static lists, exchanged once per iteration after
  the step (``ShardedGp3d``), instead of every position on every rank.
"""

from __future__ import annotations

import numpy as np


def locality_order(net_ptr, pin_inst, n_inst, sweeps=30, seed=0, device=None):
    """Permutation `perm` (new index -> old index) grouping connected
    instances (label propagation, see module docstring).  The sweeps run as
    torch sorts / scans on `device` (the current CUDA device when there is
    one: ~0.6 s at config 3 instead of ~80 s of numpy on one core); every op
    is deterministic (stable sorts, integer scans, a seeded numpy RNG), so
    every rank of a sharded run computes the same numbering."""
    import torch

    net_ptr = np.asarray(net_ptr, dtype=np.int64)
    pin_inst = np.asarray(pin_inst, dtype=np.int64)
    deg = np.diff(net_ptr)
    if n_inst == 0 or len(pin_inst) == 0:
        return np.arange(n_inst, dtype=np.int64)
    # clique expansion: (a, b, w) for every ordered pin pair of a net
    a_list, b_list, w_list = [], [], []
    for d in np.unique(deg):
        if d < 2:
            continue
        nets = np.flatnonzero(deg == d)
        base = net_ptr[nets]
        pins = pin_inst[base[:, None] + np.arange(d)[None, :]]  # [n_d, d]
        ii, jj = np.nonzero(~np.eye(d, dtype=bool))
        a_list.append(pins[:, ii].reshape(-1))
        b_list.append(pins[:, jj].reshape(-1))
        # integer weights (2^30 / (d - 1)): the segment sums below are exact
        # integer scans, identical for any scan order on any device
        w_list.append(np.full(len(nets) * len(ii), int(round((1 << 30) / (d - 1))), np.int64))
    if not a_list:
        return np.arange(n_inst, dtype=np.int64)
    a = np.concatenate(a_list)
    b = np.concatenate(b_list)
    w = np.concatenate(w_list)
    keep = a != b
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    dev = torch.device(device)
    a, b, w = (torch.from_numpy(np.ascontiguousarray(v[keep])).to(dev) for v in (a, b, w))
    n1 = n_inst + 1
    rs = np.random.default_rng(seed)
    label = torch.arange(n_inst, dtype=torch.int64, device=dev)

    def starts_of(sorted_keys):
        m = torch.ones(sorted_keys.numel(), dtype=torch.bool, device=dev)
        m[1:] = sorted_keys[1:] != sorted_keys[:-1]
        return torch.nonzero(m).squeeze(1)

    for _ in range(sweeps):
        # total weight per (instance, neighbour label): segment sums of the
        # key-sorted edge weights (differences of one inclusive scan)
        ks, order = torch.sort(a * n1 + label[b], stable=True)
        first = starts_of(ks)
        csum = torch.cumsum(w[order], 0)  # int64: exact
        last = torch.empty_like(first)
        last[:-1] = first[1:] - 1
        last[-1] = ks.numel() - 1
        tot = (csum[last] - torch.where(first > 0, csum[(first - 1).clamp(min=0)],
                                        torch.zeros((), dtype=csum.dtype, device=dev)))
        tot = tot.to(torch.float64) * 2.0 ** -30
        inst = ks[first] // n1
        lab = ks[first] % n1
        # ties broken by a random rank per label (fixed seed: deterministic)
        jitter = torch.from_numpy(rs.random(n1)).to(dev)[lab] * 1e-9
        # best label per instance: order by (instance, -weight), first of each
        o = torch.sort(-(tot + jitter), stable=True).indices
        o = o[torch.sort(inst[o], stable=True).indices]
        inst_o = inst[o]
        best = starts_of(inst_o)
        upd = inst_o[best]
        best_lab = lab[o][best]
        # semi-synchronous: a random half of the instances adopts its best
        # label per sweep (fully synchronous updates oscillate between
        # neighbouring labels)
        take = torch.from_numpy(rs.random(upd.numel()) < 0.5).to(dev)
        new = label.clone()
        new[upd[take]] = best_lab[take]
        changed = int((new != label).sum().item())
        label = new
        if changed <= n_inst // 1000:
            break
    # sort by label, ties by index (a stable sort of the labels)
    return torch.sort(label, stable=True).indices.cpu().numpy().astype(np.int64)


def cached_locality_order(net_ptr, pin_inst, n_inst, cache_dir=None):
    """locality_order with an on-disk cache keyed by the netlist (every run on
    the same box computes it once)."""
    import hashlib
    import os

    net_ptr = np.ascontiguousarray(net_ptr, dtype=np.int64)
    pin_inst = np.ascontiguousarray(pin_inst, dtype=np.int64)
    h = hashlib.sha1(net_ptr.tobytes() + pin_inst.tobytes() + str(n_inst).encode()).hexdigest()[:16]
    cache_dir = cache_dir or os.environ.get("P3D_CACHE", "/tmp/p3d_cache")
    path = os.path.join(cache_dir, f"locality2_{n_inst}_{h}.npy")
    if os.path.exists(path):
        try:
            perm = np.load(path)
            if len(perm) == n_inst:
                return perm
        except (OSError, ValueError):
            pass
    perm = locality_order(net_ptr, pin_inst, n_inst)
    try:
        os.makedirs(cache_dir, exist_ok=True)
        tmp = f"{path}.{os.getpid()}.tmp.npy"
        np.save(tmp, perm)
        os.replace(tmp, path)
    except OSError:
        pass
    return perm


class HaloPlan:
    """Per-rank net sets and position halos of the sharded loop (module
    docstring).  Instance slabs: rank r owns [r * slab, (r + 1) * slab)."""

    def __init__(self, net_ptr, pin_inst, n_inst, world, slab):
        net_ptr = np.asarray(net_ptr, dtype=np.int64)
        pin_inst = np.asarray(pin_inst, dtype=np.int64)
        self.world, self.slab, self.n_inst = int(world), int(slab), int(n_inst)
        deg = np.diff(net_ptr)
        n_net = len(deg)
        pin_net = np.repeat(np.arange(n_net), deg)
        owner = pin_inst // max(slab, 1)
        self.primary = np.full(n_net, -1, dtype=np.int64)
        has = deg > 0
        self.primary[has] = owner[net_ptr[:-1][has]]  # the owner of the net's first pin
        # touches[r]: nets with a pin in slab r
        self.touches = []
        self.halo = []
        for r in range(world):
            t = np.zeros(n_net, dtype=bool)
            t[pin_net[owner == r]] = True
            self.touches.append(t)
            pins = np.flatnonzero(t[pin_net])
            inst = np.unique(pin_inst[pins])
            self.halo.append(inst[(inst // max(slab, 1)) != r])
        # send[r][s]: instances of slab r that rank s needs (sorted)
        self.send = [[self.halo[s][(self.halo[s] // max(slab, 1)) == r] if s != r
                      else np.zeros(0, dtype=np.int64) for s in range(world)]
                     for r in range(world)]

    def nets_of(self, rank):
        """(net mask evaluated by `rank`, mask of those it counts the value of)."""
        t = self.touches[rank]
        return t, t & (self.primary == rank)

    def exchange_bytes(self, rank, bytes_per_inst=32):
        """Position bytes received per iteration by `rank` (pos4 rows)."""
        return int(len(self.halo[rank]) * bytes_per_inst)

    def split_sizes(self, rank):
        """(input splits: rows sent to each rank, output splits: rows received
        from each rank) of the all-to-all halo exchange."""
        ins = [len(self.send[rank][s]) for s in range(self.world)]
        outs = [len(self.send[s][rank]) for s in range(self.world)]
        return ins, outs


__all__ = ["HaloPlan", "cached_locality_order", "locality_order"]
