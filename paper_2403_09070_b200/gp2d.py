"""Multi-die 2D global placement (run_gp2d_multi, gp.py:463-690) on the B200.

The second GP pass of the reference flow for designs with r_MA >= 0.5
(gp.py:110-112, flow.py:110-120): the partition is frozen, the HBTs of the
crossing nets become movable objects, and three independent planar fields
(bottom die, top die, terminal layer; nz = 1 grids) are coupled only through
the wirelength.  Same signature, RNG draw order, log rows and return value as
the reference; the per-iteration work runs on the device:

* wirelength: ``p3d_gp2d_wirelength`` — the partial-net weighted-average span
  of every (net, die) segment of the augmented pin list and its owner sums;
* density per layer: the K2 fixed-point scatter, the K3 spectral solve and
  the K4 force gather of the 3D path, on an nz = 1 grid (density.py API);
* loop control (``p3d_gp2d_step``): per-layer lambda init, the log row and
  the stop test, the Eq. 19 preconditioning of the current and the
  re-weighted previous gradient, the Nesterov / BB step with the 2D span
  clamp as projection, the step-underflow exit and the per-layer mu update,
  with every scalar in a device-resident ``p3d_gp2d_state``.

One iteration is captured as a CUDA graph and replayed; the host polls the
done flag every few replays and reads the log rows once at the end.  Host
work is setup only (partition, augmented pin list, fillers with the
reference's numpy RNG stream).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _dev, _lib
from . import density as dn
from . import wirelength as wl
from .gp import GRID_SMS, GpConfig, GpInfo, gamma_schedule
from .model import partition_from_z, rotate_offsets, rotated_dims


def gp2d_grid_n(n_insts):
    """Bins per side of the three planar grids (gp.py:536-539)."""
    n = max(n_insts, 1)
    k = 2
    while (2 ** (k + 1)) ** 2 <= n / 4 and 2 ** (k + 1) <= 128:
        k += 1
    return 2 ** k


class Gp2dProblem:
    """gp.py:463-528: three nz = 1 grids, the augmented pin list in which each
    HBT joins both partial nets of its crossing net, and pin offsets frozen at
    the partition.  Device copies of the pin list are built once."""

    def __init__(self, design, cfg: GpConfig, delta, rot, n_grid):
        self.design = design
        self.cfg = cfg
        self.arr = arr = design.arrays()
        self.delta = np.asarray(delta)
        self.rot = rot
        die = design.die
        self.grids = [dn.DensityGrid(die.width, die.height, n_grid, n_grid, 1) for _ in range(3)]
        pd = self.delta[arr.pin_inst]
        mx = np.zeros(design.n_nets, dtype=np.int8)
        mn = np.ones(design.n_nets, dtype=np.int8)
        np.maximum.at(mx, arr.pin_net, pd)
        np.minimum.at(mn, arr.pin_net, pd)
        self.crossing = np.flatnonzero(mx > mn)
        self.n_inst = design.n_insts
        self.n_hbt = len(self.crossing)
        self.n_obj_core = self.n_inst + self.n_hbt
        pin_net = np.r_[arr.pin_net, self.crossing, self.crossing]
        pin_obj = np.r_[arr.pin_inst, self.n_inst + np.arange(self.n_hbt),
                        self.n_inst + np.arange(self.n_hbt)]
        top = np.r_[pd == 1, np.ones(self.n_hbt, bool), np.zeros(self.n_hbt, bool)]
        order = np.argsort(pin_net, kind="stable")
        self.pin_net, self.pin_obj, self.pin_on_top = pin_net[order], pin_obj[order], top[order]
        counts = np.bincount(self.pin_net, minlength=design.n_nets)
        self.net_ptr = np.zeros(design.n_nets + 1, dtype=np.int64)
        np.cumsum(counts, out=self.net_ptr[1:])
        wt, ht = rotated_dims(arr.w_top, arr.h_top, rot)
        wb, hb = rotated_dims(arr.w_bot, arr.h_bot, rot)
        self.inst_w = np.where(self.delta == 1, wt, wb)
        self.inst_h = np.where(self.delta == 1, ht, hb)
        self.hbt_size = design.hbt.pitch + design.hbt.spacing
        q = np.asarray(rot)[arr.pin_inst]
        rx_t, ry_t = rotate_offsets(arr.ox_top, arr.oy_top, q)
        rx_b, ry_b = rotate_offsets(arr.ox_bot, arr.oy_bot, q)
        it = pd == 1
        self.pin_ox = np.r_[np.where(it, rx_t, rx_b), np.zeros(2 * self.n_hbt)][order]
        self.pin_oy = np.r_[np.where(it, ry_t, ry_b), np.zeros(2 * self.n_hbt)][order]

    def layer_objects(self):
        """(object ids) for bottom(0) / top(1) / hbt(2) layers (gp.py:520-528)."""
        return [np.flatnonzero(self.delta == 0), np.flatnonzero(self.delta == 1),
                self.n_inst + np.arange(self.n_hbt)]

    def device_pins(self, n_obj):
        """Device pin list with owner-sorted record slots for the owner sums."""
        P = len(self.pin_obj)
        slot_order = np.argsort(self.pin_obj, kind="stable")
        pin_slot = np.empty(P, dtype=np.int64)
        pin_slot[slot_order] = np.arange(P)
        optr = np.zeros(n_obj + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.pin_obj, minlength=n_obj), out=optr[1:])
        one = lambda a, dt: a if len(a) else np.zeros(1, dt)  # noqa: E731
        return dict(
            net_ptr=_dev.i32(self.net_ptr), pin_obj=_dev.i32(one(self.pin_obj, np.int64)),
            pin_top=_dev.u8(one(self.pin_on_top, bool)), pin_ox=_dev.f64(one(self.pin_ox, float)),
            pin_oy=_dev.f64(one(self.pin_oy, float)), pin_slot=_dev.i32(one(pin_slot, np.int64)),
            obj_slot_ptr=_dev.i32(optr), n_pin=P)


def gp2d_wirelength(prob: Gp2dProblem, dp, pos_soa, n_obj, gamma):
    """(value, wl_grad [n_obj, 2]) at positions pos_soa [2][n_obj] (gp.py:586-600)."""
    value = torch.zeros(1, dtype=torch.float64, device="cuda")
    grad = torch.empty((n_obj, 2), dtype=torch.float64, device="cuda")
    scr = _dev.scratch(2 * dp["n_pin"] + 8 + 1024)
    _lib.call("p3d_gp2d_wirelength", int(len(prob.net_ptr) - 1), int(dp["n_pin"]), int(n_obj),
              _lib.ptr(dp["net_ptr"]), _lib.ptr(dp["pin_obj"]), _lib.ptr(dp["pin_top"]),
              _lib.ptr(dp["pin_ox"]), _lib.ptr(dp["pin_oy"]), _lib.ptr(dp["pin_slot"]),
              _lib.ptr(dp["obj_slot_ptr"]), _lib.ptr(pos_soa), float(gamma), _lib.ptr(value),
              _lib.ptr(grad), _lib.ptr(scr), _lib.stream_ptr())
    return value, grad


class _Layer:
    """One planar field of the 2D GP (nz = 1 grid): a persistent device charge
    cloud whose x/y buffers are refreshed from the positions each iteration,
    then the K2 scatter, the K3 spectral solve (one pass: phi and E), the K4
    force gather and the fixed-point overflow, all through the C-ABI."""

    def __init__(self, grid, idx, sw, sh, weight, is_macro, movable_volume, rho_t):
        self.grid, self.idx, self.n = grid, idx, int(idx.numel())
        self.mv, self.rho_t = movable_volume, rho_t
        if not self.n:
            return
        k = self.n
        full = lambda v: torch.full((k,), v, dtype=torch.float64, device="cuda")  # noqa: E731
        self.x = torch.empty(k, dtype=torch.float64, device="cuda")
        self.y = torch.empty(k, dtype=torch.float64, device="cuda")
        self.cloud = dn.ChargeCloud(x=self.x, y=self.y, z=full(grid.dz / 2), w=sw[idx].contiguous(),
                                    h=sh[idx].contiguous(), dep=full(grid.dz),
                                    weight=_dev.f64(weight), is_macro=np.asarray(is_macro))
        self.dc = dn._DevCloud(self.cloud)
        # the cloud's x / y are the buffers refreshed below
        self.dc.struct.x = _lib.ptr(self.x).value
        self.dc.struct.y = _lib.ptr(self.y).value
        self.g, _ = grid.device()
        B = grid.n_bins
        self.rho_fx = torch.zeros(B, dtype=torch.int64, device="cuda")
        self.maps = torch.empty((B, 4), dtype=torch.float64, device="cuda")
        self.spec = torch.empty(6 * B, dtype=torch.float64, device="cuda")
        self.force = torch.empty((k, 3), dtype=torch.float64, device="cuda")
        self.energy = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.gscr = _dev.scratch(8 + self.dc.struct.n_macro + 1024 + 8)
        self.oscr = _dev.scratch(8 + 1024 + 8)
        self.idx32 = idx.to(torch.int32).contiguous()

    def enqueue(self, pos_soa, n_obj, dens_grad, ovfl_out, halt):
        """gp.py:610-626 for this layer at pos_soa [2][n_obj] (stream-ordered)."""
        g, s = _lib.byref(self.g), _lib.stream_ptr()
        _lib.call("p3d_gp2d_layer_xy", self.n, _lib.ptr(self.idx32), _lib.ptr(pos_soa), int(n_obj),
                  _lib.ptr(self.x), _lib.ptr(self.y), _lib.ptr(halt), s)
        # rho_fx is zero here: allocated zeroed, re-zeroed by the solve that reads it
        _lib.call("p3d_accumulate_density", g, _lib.byref(self.dc.struct), _lib.ptr(self.rho_fx), s)
        # field maps straight from the fixed-point map, the overflow fused in
        _lib.call("p3d_spectral_fx", g, _lib.ptr(self.rho_fx), _lib.ptr(self.maps),
                  _lib.ptr(self.spec), float(self.rho_t), float(self.mv), _lib.ptr(ovfl_out),
                  _lib.ptr(self.oscr), 1, s)
        _lib.call("p3d_density_gather", g, _lib.byref(self.dc.struct), _lib.ptr(self.maps), None,
                  _lib.ptr(self.energy), _lib.ptr(self.force), _lib.ptr(self.gscr), s)
        _lib.call("p3d_gp2d_layer_force", self.n, _lib.ptr(self.idx32), _lib.ptr(self.force),
                  _lib.ptr(dens_grad), _lib.ptr(halt), s)


class Gp2dLoop:
    """The device-resident iteration of run_gp2d_multi (gp.py:640-681): the
    wirelength, the three layers and ``p3d_gp2d_step`` enqueued on one stream
    (graph-capturable); every loop scalar lives in ``p3d_gp2d_state``."""

    def __init__(self, prob, dp, layers, n_obj, size_w, size_h, obj_layer, is_macro_obj,
                 degree_obj, charges, grid0, cfg, die):
        self.prob, self.dp, self.layers, self.n_obj = prob, dp, layers, n_obj
        keep = self._keep = _dev.Keep()
        mi = max(int(cfg.max_iters), 1)
        z = lambda n: torch.zeros(max(int(n), 1), dtype=torch.float64, device="cuda")  # noqa: E731
        self.u, self.v = z(2 * n_obj), z(2 * n_obj)
        self.wl_grad, self.dens_grad = z(2 * n_obj), z(2 * n_obj)
        self.prev_wl, self.prev_dens, self.pre = z(2 * n_obj), z(2 * n_obj), z(2 * n_obj)
        self.value, self.ovfl = z(1), z(3)
        self.log = z(4 * mi)
        self.wl_scr = _dev.scratch(2 * dp["n_pin"] + 8 + 1024)
        self.st = torch.zeros(C.sizeof(_lib.Gp2dState), dtype=torch.uint8, device="cuda")
        self._st_host = torch.empty(C.sizeof(_lib.Gp2dState), dtype=torch.uint8, pin_memory=True)
        n_sm = GRID_SMS  # fixed: the block count partitions its reductions (gp.GRID_SMS)
        c = self.ctl = _lib.Gp2dCtl()
        c.n_obj, c.max_iters, c.n_hbt = int(n_obj), int(cfg.max_iters), int(prob.n_hbt)
        c.nblk = max(1, min(-(-max(n_obj, 1) // 256), 2 * n_sm, 2048))
        c.layer = keep(_dev.i32(obj_layer))
        c.size_w, c.size_h = keep(_dev.f64(size_w)), keep(_dev.f64(size_h))
        c.charge = keep(_dev.f64(charges))
        c.is_macro = keep(_dev.u8(is_macro_obj))
        c.degree = keep(_dev.f64(degree_obj))
        gam = [gamma_schedule(grid0, it, cfg.max_iters, cfg) for it in range(mi)]
        c.gamma_tab = keep(_dev.f64(np.asarray(gam, dtype=np.float64)))
        c.die_w, c.die_h = float(die.width), float(die.height)
        c.stop_overflow, c.mu_min, c.mu_max = cfg.stop_overflow, cfg.mu_min, cfg.mu_max
        c.step_scale, c.min_step = grid0.wb, 1e-18
        for name in ("u", "v", "wl_grad", "dens_grad", "prev_wl", "prev_dens", "pre", "log"):
            setattr(c, name, keep(getattr(self, name)))
        c.wl_value, c.ovfl = keep(self.value), keep(self.ovfl)
        c.partials = keep(_dev.scratch(8 * c.nblk + 8))
        c.st = keep(self.st)
        # p3d_gp2d_state field offsets of gamma / done (the WL kernel and the
        # layer kernels read them straight from device memory)
        self.gamma_ptr = self.st[_lib.Gp2dState.gamma.offset:].view(torch.float64)[:1] \
            if _lib.Gp2dState.gamma.offset % 8 == 0 else None
        self.halt = self.st[_lib.Gp2dState.done.offset:].view(torch.int32)[:1]

    def state(self):
        self._st_host.copy_(self.st)
        return _lib.Gp2dState.from_buffer_copy(bytes(self._st_host.numpy()))

    def init(self, pos0_soa):
        _lib.call("p3d_gp2d_init", _lib.byref(self.ctl), _lib.ptr(pos0_soa), _lib.stream_ptr())

    def iterate(self):
        """One iteration (gp.py:641-681), stream-ordered, no host sync.  The
        three layers' fields are independent of each other and of the
        wirelength: each runs on its own side stream (concurrent branches
        of the captured graph), joined before the step."""
        dp, n_obj = self.dp, self.n_obj
        main = torch.cuda.current_stream()
        if not hasattr(self, "_side"):
            self._side = [torch.cuda.Stream() for _ in self.layers]
        for layer, (ctx, side) in enumerate(zip(self.layers, self._side)):
            if ctx.n:
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    ctx.enqueue(self.v, n_obj, self.dens_grad, self.ovfl[layer:layer + 1],
                                self.halt)
        _lib.call("p3d_gp2d_wirelength_ex", int(len(self.prob.net_ptr) - 1), int(dp["n_pin"]),
                  int(n_obj), _lib.ptr(dp["net_ptr"]), _lib.ptr(dp["pin_obj"]),
                  _lib.ptr(dp["pin_top"]), _lib.ptr(dp["pin_ox"]), _lib.ptr(dp["pin_oy"]),
                  _lib.ptr(dp["pin_slot"]), _lib.ptr(dp["obj_slot_ptr"]), _lib.ptr(self.v),
                  _lib.ptr(self.gamma_ptr), _lib.ptr(self.halt), _lib.ptr(self.value),
                  _lib.ptr(self.wl_grad), _lib.ptr(self.wl_scr), _lib.stream_ptr())
        for ctx, side in zip(self.layers, self._side):
            if ctx.n:
                main.wait_stream(side)
        _lib.call("p3d_gp2d_step", _lib.byref(self.ctl), _lib.stream_ptr())

    def capture(self):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            self.iterate()
        torch.cuda.current_stream().wait_stream(s)
        return g

    def run(self, pos0_soa, use_graph=True, poll_every=8):
        self.init(pos0_soa)
        total = int(self.ctl.max_iters)
        if use_graph and total > 0:
            self.iterate()  # warm-up outside capture (first-use allocations)
            self.init(pos0_soa)
            g = self.capture()
            for r in range(total):
                g.replay()
                if (r + 1) % poll_every == 0 and self.state().done:
                    break
        else:
            for r in range(total):
                self.iterate()
                if (r + 1) % poll_every == 0 and self.state().done:
                    break
        return self.state()

    def log_rows(self, n):
        rows = self.log[: 4 * n].reshape(n, 4).cpu().numpy()
        return [(int(r[0]), float(r[1]), int(r[2]), float(r[3])) for r in rows]

    def project(self, soa):
        out = torch.empty_like(soa)
        _lib.call("p3d_gp2d_project", _lib.byref(self.ctl), _lib.ptr(soa), _lib.ptr(out),
                  _lib.stream_ptr())
        return out


def run_gp2d_multi(design, state, cfg: GpConfig, iteration_log=None, rng=None, use_graph=True):
    """Planar refinement with a fixed partition (gp.py:531-690); returns
    (state, GpInfo, {crossing net: HBT centre}).  use_graph (not in the
    reference signature): replay one captured iteration (default) or enqueue
    each iteration eagerly."""
    rng = rng or np.random.default_rng(cfg.seed)
    loop, pos0 = setup_gp2d(design, state, cfg, rng)
    prob, n_obj = loop.prob, loop.n_obj
    st = loop.run(pos0, use_graph=use_graph)
    info = GpInfo(iterations=int(st.iterations), final_overflow=float(st.final_overflow),
                  diverged=bool(st.diverged))
    if iteration_log is not None:
        iteration_log.extend(loop.log_rows(int(st.iterations)))
    final = loop.project(loop.u).reshape(2, n_obj).t().cpu().numpy()
    state.x = final[: prob.n_inst, 0].copy()
    state.y = final[: prob.n_inst, 1].copy()
    hbt_centers = {int(j): (float(final[prob.n_inst + t, 0]), float(final[prob.n_inst + t, 1]))
                   for t, j in enumerate(prob.crossing)}
    return state, info, hbt_centers


def setup_gp2d(design, state, cfg: GpConfig, rng):
    """Host setup of run_gp2d_multi (gp.py:531-639, the reference's RNG draws):
    returns (Gp2dLoop, initial positions [2][n_obj] on the device)."""
    _lib.require_cuda()
    delta = partition_from_z(state.z, state.dz)
    prob = Gp2dProblem(design, cfg, delta, state.rot, gp2d_grid_n(design.n_insts))
    die = design.die
    grids = prob.grids
    # fillers per die layer (gp.py:545-562; the reference's numpy RNG order)
    arrs = prob.arr
    cells = ~arrs.is_macro
    hint = float(np.median(arrs.w_bot[cells] * arrs.h_bot[cells])) if cells.any() \
        else (die.width / 32) ** 2
    fill_xy, fill_wh, fill_layer = [], [], []
    for layer, u in ((0, die.max_util_bottom), (1, die.max_util_top)):
        area = die.width * die.height * (1 - u)
        if area <= 0:
            continue
        count = int(np.clip(round(area / max(hint, 1e-9)), 1, 20000))
        side = math.sqrt(area / count)
        fill_xy.append(np.c_[rng.uniform(side / 2, die.width - side / 2, count),
                             rng.uniform(side / 2, die.height - side / 2, count)])
        fill_wh.append(np.full((count, 2), side))
        fill_layer.append(np.full(count, layer))
    fx = np.concatenate(fill_xy) if fill_xy else np.zeros((0, 2))
    fwh = np.concatenate(fill_wh) if fill_wh else np.zeros((0, 2))
    flayer = np.concatenate(fill_layer) if fill_layer else np.zeros(0, int)
    n_core = prob.n_obj_core
    n_obj = n_core + len(fx)
    pos = np.zeros((n_obj, 2))
    pos[: prob.n_inst] = np.c_[state.x, state.y]
    centers = wl.optimal_hbt_centers(arrs, state.x, state.y, state.z, state.rot, state.dz)
    for t, j in enumerate(prob.crossing):
        pos[prob.n_inst + t] = centers.get(int(j), (die.width / 2, die.height / 2))
    pos[n_core:] = fx
    size_w = np.r_[prob.inst_w, np.full(prob.n_hbt, prob.hbt_size), fwh[:, 0]]
    size_h = np.r_[prob.inst_h, np.full(prob.n_hbt, prob.hbt_size), fwh[:, 1]]
    obj_layer = np.r_[delta.astype(int), np.full(prob.n_hbt, 2), flayer]
    is_macro_obj = np.r_[arrs.is_macro, np.zeros(prob.n_hbt + len(fx), bool)]
    degree_obj = np.r_[arrs.pin_degree, np.full(prob.n_hbt, 2.0), np.zeros(len(fx))]
    is_filler = np.r_[np.zeros(n_core, bool), np.ones(len(fx), bool)]
    movable_vol = [float((size_w[m] * size_h[m]).sum() * grids[l].db)
                   for l, m in enumerate([(obj_layer == l) & ~is_filler for l in range(3)])]
    charges = size_w * size_h * grids[0].db

    dp = prob.device_pins(n_obj)
    sw, sh = _dev.f64(size_w), _dev.f64(size_h)
    layer_idx = [torch.from_numpy(np.flatnonzero(obj_layer == l)).cuda() for l in range(3)]
    layers = [_Layer(grids[l], layer_idx[l], sw, sh,
                     np.where(is_macro_obj[obj_layer == l], cfg.target_density, 1.0),
                     is_macro_obj[obj_layer == l], movable_vol[l], cfg.target_density)
              for l in range(3)]
    loop = Gp2dLoop(prob, dp, layers, n_obj, size_w, size_h, obj_layer, is_macro_obj,
                    degree_obj, charges, grids[0], cfg, die)
    return loop, _dev.f64(pos).t().contiguous()


__all__ = ["Gp2dProblem", "Gp2dLoop", "gp2d_grid_n", "gp2d_wirelength", "run_gp2d_multi",
           "setup_gp2d"]
