"""Fixture builders of the reference's own unit tests (pkg/tests/conftest.py,
pkg/tests/test_wirelength.py:11-18, pkg/tests/test_density.py:10-45),
restated over this package's types so the restated suites
(test_reference_suite_host.py, test_gpu_reference_suite.py) need no reference
import at run time.  Test infrastructure only."""

from __future__ import annotations

import numpy as np

from paper_2403_09070_b200 import density as dn
from paper_2403_09070_b200 import wirelength as wl
from paper_2403_09070_b200.model import ArrayDesign, DieSpec, HbtSpec, NetlistArrays


class Kind:
    """conftest.py:8-15 make_kind: a cell kind, pins by name -> (ox, oy)."""

    def __init__(self, name, w, h, pins):
        self.name, self.width, self.height = name, float(w), float(h)
        self.pins = {p[0]: (float(p[1]), float(p[2])) for p in pins}


def make_kind(name, w, h, pins):
    return Kind(name, w, h, pins)


def make_design(kinds_top, kinds_bot, insts, nets, *, die=(1000, 960), rows=(32, 48),
                util=(0.8, 0.8), hbt=(8, 2, 10.0)):
    """conftest.py:18-32 make_design, straight to the flat arrays the
    reference's NetlistArrays (model.py:231-275) derives from a Design:
    per-die kind dims, per-die pin offsets looked up by pin name."""
    top = {k.name: k for k in kinds_top}
    bot = {k.name: k for k in kinds_bot}
    kinds = [i[1] for i in insts]
    counts = [len(p) for _, p in nets]
    net_ptr = np.zeros(len(nets) + 1, dtype=np.int64)
    np.cumsum(counts, out=net_ptr[1:])
    pins = [pp for _, p in nets for pp in p]
    arrays = NetlistArrays(
        is_macro=[bool(i[2]) for i in insts],
        w_top=[top[k].width for k in kinds], h_top=[top[k].height for k in kinds],
        w_bot=[bot[k].width for k in kinds], h_bot=[bot[k].height for k in kinds],
        net_ptr=net_ptr, pin_inst=np.array([p[0] for p in pins], dtype=np.int64),
        ox_top=[top[kinds[i]].pins[n][0] for i, n in pins],
        oy_top=[top[kinds[i]].pins[n][1] for i, n in pins],
        ox_bot=[bot[kinds[i]].pins[n][0] for i, n in pins],
        oy_bot=[bot[kinds[i]].pins[n][1] for i, n in pins])
    return ArrayDesign(DieSpec(float(die[0]), float(die[1]), float(rows[0]), float(rows[1]),
                               float(util[0]), float(util[1])),
                       HbtSpec(float(hbt[0]), float(hbt[1]), float(hbt[2])), arrays)


def random_net(rng, n_pins, span=100, allow_empty_side=True):
    """conftest.py:47-57: (coords, on_top) with possible boundary ties."""
    base = rng.integers(0, span, n_pins).astype(float)
    if n_pins >= 2 and rng.random() < 0.4:
        base[rng.integers(0, n_pins)] = base.max()
    on_top = rng.random(n_pins) < rng.uniform(0.1, 0.9)
    if not allow_empty_side and (on_top.all() or not on_top.any()):
        on_top[0] = ~on_top[0]
    return base, on_top


def make_topo(nets):
    """test_wirelength.py:11-18: one distinct owner per pin."""
    ptr = np.zeros(len(nets) + 1, dtype=np.int64)
    np.cumsum(nets, out=ptr[1:])
    n_pin = int(ptr[-1])
    return wl.NetTopology(ptr, np.repeat(np.arange(len(nets)), nets), np.arange(n_pin), n_pin)


def make_cloud(boxes, weights=None, macro=None):
    """test_density.py:10-19: boxes are (x, y, z, w, h, dep) rows."""
    b = np.asarray(boxes, dtype=float).reshape(-1, 6)
    n = len(b)
    return dn.ChargeCloud(
        x=b[:, 0].copy(), y=b[:, 1].copy(), z=b[:, 2].copy(), w=b[:, 3].copy(),
        h=b[:, 4].copy(), dep=b[:, 5].copy(),
        weight=np.ones(n) if weights is None else np.asarray(weights, float),
        is_macro=np.zeros(n, bool) if macro is None else np.asarray(macro, bool))


def brute_density(grid, cloud):
    """test_density.py:22-45: triple-loop overlap integration."""
    rho = np.zeros(grid.shape)
    for i in range(len(cloud.x)):
        lo = (max(cloud.x[i] - cloud.w[i] / 2, 0.0), max(cloud.y[i] - cloud.h[i] / 2, 0.0),
              max(cloud.z[i] - cloud.dep[i] / 2, 0.0))
        hi = (min(cloud.x[i] + cloud.w[i] / 2, grid.dx), min(cloud.y[i] + cloud.h[i] / 2, grid.dy),
              min(cloud.z[i] + cloud.dep[i] / 2, grid.dz))
        for bx in range(grid.nx):
            ox = min(hi[0], (bx + 1) * grid.wb) - max(lo[0], bx * grid.wb)
            if ox <= 0:
                continue
            for by in range(grid.ny):
                oy = min(hi[1], (by + 1) * grid.hb) - max(lo[1], by * grid.hb)
                if oy <= 0:
                    continue
                for bz in range(grid.nz):
                    oz = min(hi[2], (bz + 1) * grid.db) - max(lo[2], bz * grid.db)
                    if oz > 0:
                        rho[bx, by, bz] += cloud.weight[i] * ox * oy * oz / grid.bin_vol
    return rho
