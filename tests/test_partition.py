"""Host side of the sharded loop's halo mode (paper_2403_09070_b200.partition,
SURVEY 8e), on CPU:

* the locality numbering is a permutation that makes the synthetic netlist's
  clusters contiguous: far fewer nets cross instance slabs than in the
  generator's random numbering;
* the halo plan evaluates every net on every rank it touches, counts each
  net's value on exactly one rank, gives each rank the positions of exactly
  the remote pins of its nets, and its send / receive lists pair up;
* the exchanged bytes per iteration are a fraction of the round-robin mode's
  (owner-sum reduce-scatter + full position all-gather).
"""

import numpy as np
import pytest

from paper_2403_09070_b200.dist import object_slabs
from paper_2403_09070_b200.partition import HaloPlan, locality_order
from paper_2403_09070_b200.synth import SynthSpec, synth_arrays


@pytest.fixture(scope="module")
def design():
    return synth_arrays(SynthSpec(n_insts=20_000, n_macros=8, r_ma=0.3, seed=1, nets_per_inst=1.1))


def _crossing_fraction(net_ptr, pin_inst, slab):
    owner = pin_inst // slab
    deg = np.diff(net_ptr)
    pin_net = np.repeat(np.arange(len(deg)), deg)
    mx = np.full(len(deg), -1)
    mn = np.full(len(deg), 1 << 30)
    np.maximum.at(mx, pin_net, owner)
    np.minimum.at(mn, pin_net, owner)
    return float(np.mean(mx > mn))


def test_locality_order_is_a_permutation_and_local(design):
    a = design.arrays()
    I = design.n_insts
    perm = locality_order(a.net_ptr, a.pin_inst, I)
    assert np.array_equal(np.sort(perm), np.arange(I))
    inv = np.empty_like(perm)
    inv[perm] = np.arange(I)
    slab = -(-I // 8)
    before = _crossing_fraction(a.net_ptr, a.pin_inst, slab)
    after = _crossing_fraction(a.net_ptr, inv[a.pin_inst], slab)
    assert before > 0.8  # random numbering: almost every net crosses 8 slabs
    assert after < 0.35, after  # ~80% of the generator's nets are intra-cluster
    assert np.array_equal(perm, locality_order(a.net_ptr, a.pin_inst, I))  # deterministic


@pytest.mark.parametrize("world", [2, 3, 8])
def test_halo_plan_invariants(design, world):
    a = design.arrays()
    I = design.n_insts
    perm = locality_order(a.net_ptr, a.pin_inst, I)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(I)
    pin_inst = inv[a.pin_inst]
    slab, _, _ = object_slabs(I, 0, 0, world)
    plan = HaloPlan(a.net_ptr, pin_inst, I, world, slab)
    deg = np.diff(a.net_ptr)
    pin_net = np.repeat(np.arange(len(deg)), deg)
    owner = pin_inst // slab
    counted = np.zeros(len(deg), dtype=int)
    for r in range(world):
        mask, prim = plan.nets_of(r)
        # every net with a pin in slab r runs on r; nothing else does
        want = np.zeros(len(deg), bool)
        want[pin_net[owner == r]] = True
        assert np.array_equal(mask, want)
        counted += prim
        # the halo is exactly the remote instances of r's nets
        need = np.unique(pin_inst[mask[pin_net]])
        assert np.array_equal(plan.halo[r], need[need // slab != r])
        ins, outs = plan.split_sizes(r)
        assert sum(outs) == len(plan.halo[r])
        for s in range(world):
            assert np.all(plan.send[r][s] // slab == r)
            assert set(plan.send[r][s]) <= set(plan.halo[s])
    assert np.all(counted[deg > 0] == 1)  # each net's value counted exactly once
    for s in range(world):  # the halo is fully covered by the owners' send lists
        got = np.sort(np.concatenate([plan.send[r][s] for r in range(world)]))
        assert np.array_equal(got, plan.halo[s])


def test_exchange_bytes_vs_round_robin(design):
    a = design.arrays()
    I = design.n_insts
    world = 8
    perm = locality_order(a.net_ptr, a.pin_inst, I)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(I)
    slab = -(-I // world)
    plan = HaloPlan(a.net_ptr, inv[a.pin_inst], I, world, slab)
    halo = max(plan.exchange_bytes(r) for r in range(world))
    rr = 2 * 32 * slab * world  # owner-sum reduce-scatter + position all-gather
    assert halo <= 0.3 * rr, (halo, rr)
