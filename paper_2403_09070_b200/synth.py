"""Synthetic netlists straight to flat arrays (the benchmark input path).

The reference generates a text file (``place3d/synth.py:49-173``) which is then
parsed (``model.py:423-571``) and flattened (``model.py:224-275``).  At 800k
instances that chain takes ~110 s on one core, dominated by an
O(clusters x instances) grouping (``synth.py:147``) and per-pin Python loops.

``synth_arrays`` draws from the same ``numpy.random.default_rng(seed)`` stream
in the same order, so the resulting ``NetlistArrays`` are identical to
``parse_design(gen_synthetic(spec)).arrays()`` (checked against golden
checksums in ``tests/test_synth.py``), but it groups clusters with one stable
argsort and never builds text.  ``SynthSpec`` keeps the reference's field names
and defaults (``synth.py:24-40``).
"""

from __future__ import annotations

import math
import os
from dataclasses import asdict, dataclass

import numpy as np

from .model import ArrayDesign, DieSpec, HbtSpec, NetlistArrays


class InfeasibleSpec(ValueError):
    pass


@dataclass
class SynthSpec:
    n_insts: int = 100
    n_macros: int = 2
    r_ma: float = 0.3
    seed: int = 0
    row_top: int = 33
    row_bot: int = 48
    util_top: float = 0.8
    util_bot: float = 0.8
    hbt_pitch: int = 16
    hbt_spacing: int = 4
    beta: float = 10.0
    nets_per_inst: float = 1.3
    fill_fraction: float = 0.62
    local_net_fraction: float = 0.8


def _offsets(rng, w, h, n):
    ox = rng.integers(-(int(w) // 2), int(w) // 2 + 1, n)
    oy = rng.integers(-(int(h) // 2), int(h) // 2 + 1, n)
    return ox, oy


def synth_arrays(spec: SynthSpec) -> ArrayDesign:
    if spec.n_macros > spec.n_insts:
        raise InfeasibleSpec("more macros than instances")
    if not 0 <= spec.r_ma < 1:
        raise InfeasibleSpec("macro area ratio must be in [0, 1)")
    rng = np.random.default_rng(spec.seed)
    n_cells = spec.n_insts - spec.n_macros

    # library: (top w, top h, top ox, top oy, bot w, bot h, bot ox, bot oy, n_pins)
    lib = []
    n_kinds = min(6, max(1, n_cells)) if n_cells else 1
    for _ in range(n_kinds):
        wb = int(rng.integers(4, 19))
        hb = spec.row_bot
        wt = max(2, int(round(wb * (spec.row_top / spec.row_bot) * rng.uniform(0.9, 1.15))))
        ht = spec.row_top
        npin = int(rng.integers(2, 5))
        obx, oby = _offsets(rng, wb, hb, npin)
        otx, oty = _offsets(rng, wt, ht, npin)
        lib.append((wt, ht, otx, oty, wb, hb, obx, oby, npin))

    kind_of_cell = rng.integers(0, n_kinds, n_cells) if n_cells else np.zeros(0, np.int64)
    kind_area = np.array([k[4] * k[5] for k in lib], dtype=np.int64)
    cell_area = float(kind_area[kind_of_cell].sum()) if n_cells else 0.0

    capacity = spec.fill_fraction * (spec.util_top + spec.util_bot)
    if spec.r_ma >= capacity:
        raise InfeasibleSpec(f"macro ratio {spec.r_ma} beyond utilization capacity {capacity:.2f}")
    area = cell_area / max(capacity - spec.r_ma, 0.02) if cell_area else 4e5
    lcm = spec.row_top * spec.row_bot // math.gcd(spec.row_top, spec.row_bot)
    dy = max(lcm, int(round(math.sqrt(area) / lcm)) * lcm)
    dx = max(64, int(math.ceil(area / dy)))
    if dx < dy // 2:
        dx = dy // 2
    area = dx * dy

    macros = []
    if spec.n_macros:
        m_area = spec.r_ma * area / spec.n_macros
        lims = (0.45 * min(dx, dy), 0.8 * min(dx, dy))
        for _ in range(spec.n_macros):
            aspect = rng.uniform(0.6, 1.7)
            wb = max(8, int(round(math.sqrt(m_area * aspect))))
            for lim in lims:
                w_try = min(wb, int(lim))
                h_try = max(8, int(round(m_area / w_try)))
                if h_try <= lim:
                    wb, hb = w_try, h_try
                    break
            else:
                raise InfeasibleSpec("macro footprint too large to pack")
            st = rng.uniform(0.85, 1.2)
            wt = max(8, int(round(wb * st)))
            ht = max(8, int(round(hb * st)))
            npin = int(rng.integers(8, 17))
            obx, oby = _offsets(rng, wb, hb, npin)
            otx, oty = _offsets(rng, wt, ht, npin)
            macros.append((wt, ht, otx, oty, wb, hb, obx, oby, npin))
        cap = min(spec.util_top, spec.util_bot) * area
        if max(m[4] * m[5] for m in macros) > cap:
            raise InfeasibleSpec("a single macro exceeds one die's capacity")

    # per-instance kind table: cells use lib[kind], macro m uses macros[m]
    kinds = lib + macros
    inst_kind = np.concatenate([kind_of_cell.astype(np.int64),
                                n_kinds + np.arange(spec.n_macros, dtype=np.int64)])
    n_pins_of_kind = np.array([k[8] for k in kinds], dtype=np.int64)
    inst_npins = n_pins_of_kind[inst_kind]

    # nets: same draw order as synth.py:142-167
    n_insts = spec.n_insts
    n_nets = max(1, int(round(spec.nets_per_inst * n_insts)))
    deg_choices = np.array([2, 2, 2, 2, 2, 3, 3, 4, 5, 6])
    n_clusters = max(1, n_insts // 40)
    cluster_of = rng.integers(0, n_clusters, n_insts)
    by_cluster = np.argsort(cluster_of, kind="stable")
    bounds = np.zeros(n_clusters + 1, dtype=np.int64)
    np.cumsum(np.bincount(cluster_of, minlength=n_clusters), out=bounds[1:])

    integers, random, choice = rng.integers, rng.random, rng.choice
    local = spec.local_net_fraction
    npins_list = inst_npins.tolist()
    net_sizes = []
    flat_inst = []
    flat_pin = []
    for j in range(n_nets):
        deg = min(int(deg_choices[integers(0, 10)]), n_insts)
        c = int(integers(0, n_clusters))
        lo, hi = int(bounds[c]), int(bounds[c + 1])
        if random() < local and hi - lo >= deg:
            members = by_cluster[lo + choice(hi - lo, size=deg, replace=False)]
        else:
            members = choice(n_insts, size=deg, replace=False)
        if j < spec.n_macros and n_insts > spec.n_macros:
            if (n_cells + j) not in members:
                members[0] = n_cells + j
        owners = sorted(set(members.tolist()))
        pins = [int(integers(0, npins_list[i])) for i in owners]
        if len(owners) < 2:
            continue
        net_sizes.append(len(owners))
        flat_inst.extend(owners)
        flat_pin.extend(pins)

    net_ptr = np.zeros(len(net_sizes) + 1, dtype=np.int64)
    np.cumsum(net_sizes, out=net_ptr[1:])
    pin_inst = np.asarray(flat_inst, dtype=np.int64)
    pin_idx = np.asarray(flat_pin, dtype=np.int64)

    # offset tables [kind, pin] (padded), then gather
    maxp = int(n_pins_of_kind.max())
    tabs = np.zeros((4, len(kinds), maxp))
    for k, kd in enumerate(kinds):
        n = kd[8]
        tabs[0, k, :n] = kd[2]
        tabs[1, k, :n] = kd[3]
        tabs[2, k, :n] = kd[6]
        tabs[3, k, :n] = kd[7]
    pk = inst_kind[pin_inst]
    ox_top, oy_top, ox_bot, oy_bot = (tabs[t, pk, pin_idx] for t in range(4))

    geom = np.array([[k[0], k[1], k[4], k[5]] for k in kinds], dtype=np.float64)
    g = geom[inst_kind]
    is_macro = np.zeros(n_insts, dtype=bool)
    is_macro[n_cells:] = True
    arrays = NetlistArrays(
        is_macro=is_macro, w_top=g[:, 0], h_top=g[:, 1], w_bot=g[:, 2], h_bot=g[:, 3],
        net_ptr=net_ptr, pin_inst=pin_inst,
        ox_top=ox_top, oy_top=oy_top, ox_bot=ox_bot, oy_bot=oy_bot,
    )
    die = DieSpec(float(dx), float(dy), float(spec.row_top), float(spec.row_bot),
                  float(spec.util_top), float(spec.util_bot))
    hbt = HbtSpec(float(spec.hbt_pitch), float(spec.hbt_spacing), float(spec.beta))
    return ArrayDesign(die, hbt, arrays, name=f"synth{spec.n_insts}s{spec.seed}")


# --------------------------------------------------------------------------
# the BASELINE.json configurations
# --------------------------------------------------------------------------

CONFIGS = {
    1: dict(spec=SynthSpec(n_insts=10_008, n_macros=8, r_ma=0.30, seed=1, nets_per_inst=1.2), grid=128),
    2: dict(spec=SynthSpec(n_insts=100_032, n_macros=32, r_ma=0.30, seed=1, nets_per_inst=1.1), grid=256),
    3: dict(spec=SynthSpec(n_insts=800_064, n_macros=64, r_ma=0.30, seed=1, nets_per_inst=1.0625), grid=512),
    4: dict(spec=SynthSpec(n_insts=4_000_128, n_macros=128, r_ma=0.30, seed=1, nets_per_inst=1.05), grid=1024),
}


def cached_synth(spec: SynthSpec, cache_dir=None) -> ArrayDesign:
    """``synth_arrays`` with an on-disk npz cache (setup of config 3 is ~25 s)."""
    if cache_dir is None:
        # outside the repo: the snapshot shipped to the GPU box must stay small
        cache_dir = os.environ.get("P3D_CACHE", "/tmp/p3d_cache")
    key = "|".join(f"{k}={v}" for k, v in sorted(asdict(spec).items()))
    import hashlib
    h = hashlib.sha1(key.encode()).hexdigest()[:12]
    path = os.path.join(cache_dir, f"synth_{spec.n_insts}_{h}.npz")
    if os.path.exists(path):
        z = np.load(path)
        arrays = NetlistArrays(
            is_macro=z["is_macro"], w_top=z["w_top"], h_top=z["h_top"], w_bot=z["w_bot"],
            h_bot=z["h_bot"], net_ptr=z["net_ptr"], pin_inst=z["pin_inst"],
            ox_top=z["ox_top"], oy_top=z["oy_top"], ox_bot=z["ox_bot"], oy_bot=z["oy_bot"])
        d = z["die"]
        hb = z["hbt"]
        return ArrayDesign(DieSpec(*[float(v) for v in d]), HbtSpec(*[float(v) for v in hb]),
                           arrays, name=str(z["name"]))
    des = synth_arrays(spec)
    a = des.arrays()
    try:
        os.makedirs(cache_dir, exist_ok=True)
        tmp = f"{path}.{os.getpid()}.tmp.npz"  # per process: ranks may race here
        np.savez(tmp, is_macro=a.is_macro, w_top=a.w_top, h_top=a.h_top, w_bot=a.w_bot,
                 h_bot=a.h_bot, net_ptr=a.net_ptr, pin_inst=a.pin_inst, ox_top=a.ox_top,
                 oy_top=a.oy_top, ox_bot=a.ox_bot, oy_bot=a.oy_bot,
                 die=np.array([des.die.width, des.die.height, des.die.row_height_top,
                               des.die.row_height_bottom, des.die.max_util_top,
                               des.die.max_util_bottom]),
                 hbt=np.array([des.hbt.pitch, des.hbt.spacing, des.hbt.cost]),
                 name=np.array(des.name))
        os.replace(tmp, path)
    except OSError:
        pass
    return des
