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
* preconditioner (Eq. 19) and the Nesterov / BB step of the drop-in
  ``NesterovOptimizer`` with the 2D span clamp as projection.

Host work is setup only (partition, augmented pin list, fillers with the
reference's numpy RNG stream) plus one overflow scalar read per iteration for
the stop test, as in the reference loop.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _dev, _lib
from . import density as dn
from . import wirelength as wl
from .gp import (GpConfig, GpInfo, NesterovOptimizer, StepUnderflow, gamma_schedule,
                 lambda_init, mu_from_overflow, precondition)
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
        self.g, _ = grid.device()
        B = grid.n_bins
        self.rho_fx = torch.zeros(B, dtype=torch.int64, device="cuda")
        self.rho = torch.empty(B, dtype=torch.float64, device="cuda")
        self.maps = torch.empty((B, 4), dtype=torch.float64, device="cuda")
        self.spec = torch.empty(6 * B, dtype=torch.float64, device="cuda")
        self.force = torch.empty((k, 3), dtype=torch.float64, device="cuda")
        self.energy = torch.zeros(1, dtype=torch.float64, device="cuda")
        self.gscr = _dev.scratch(8 + self.dc.struct.n_macro + 1024 + 8)
        self.oscr = _dev.scratch(8 + 1024 + 8)

    def run(self, p, dens_grad, ovfl_out):
        torch.index_select(p[:, 0], 0, self.idx, out=self.x)
        torch.index_select(p[:, 1], 0, self.idx, out=self.y)
        g, s = _lib.byref(self.g), _lib.stream_ptr()
        self.rho_fx.zero_()
        _lib.call("p3d_accumulate_density", g, _lib.byref(self.dc.struct), _lib.ptr(self.rho_fx), s)
        _lib.call("p3d_fx_to_density", int(self.rho.numel()), _lib.ptr(self.rho_fx),
                  _lib.ptr(self.rho), s)
        _lib.call("p3d_spectral", g, _lib.ptr(self.rho), None, _lib.ptr(self.maps),
                  _lib.ptr(self.spec), s)
        _lib.call("p3d_density_gather", g, _lib.byref(self.dc.struct), _lib.ptr(self.maps), None,
                  _lib.ptr(self.energy), _lib.ptr(self.force), _lib.ptr(self.gscr), s)
        dens_grad[self.idx] = self.force[:, :2]
        _lib.call("p3d_overflow_fx", g, _lib.ptr(self.rho_fx), float(self.rho_t), float(self.mv),
                  _lib.ptr(ovfl_out), _lib.ptr(self.oscr), s)


def run_gp2d_multi(design, state, cfg: GpConfig, iteration_log=None, rng=None):
    """Planar refinement with a fixed partition (gp.py:531-690); returns
    (state, GpInfo, {crossing net: HBT centre})."""
    _lib.require_cuda()
    rng = rng or np.random.default_rng(cfg.seed)
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

    # ---- device constants
    dp = prob.device_pins(n_obj)
    sw, sh = _dev.f64(size_w), _dev.f64(size_h)

    def bounds(size, extent):  # gp.py:344-348 per object
        lo, hi = size / 2, extent - size / 2
        return torch.minimum(lo, hi), torch.maximum(lo, hi), lo <= hi, \
            torch.minimum(lo, hi) + (hi - lo).abs() / 2

    bx, by = bounds(sw, die.width), bounds(sh, die.height)

    def project(p):
        out = p.clone()
        for c, (lo, hi, ok, mid) in ((0, bx), (1, by)):
            out[:, c] = torch.where(ok, torch.minimum(torch.maximum(p[:, c], lo), hi), mid)
        return out

    layer_idx = [torch.from_numpy(np.flatnonzero(obj_layer == l)).cuda() for l in range(3)]
    layers = [_Layer(grids[l], layer_idx[l], sw, sh,
                     np.where(is_macro_obj[obj_layer == l], cfg.target_density, 1.0),
                     is_macro_obj[obj_layer == l], movable_vol[l], cfg.target_density)
              for l in range(3)]

    def evaluate(p, gamma):
        """gp.py:586-626: WL value/grads + per-layer raw density grads/overflow
        (one host read per iteration: the WL value and the three overflows)."""
        pos_soa = p.t().contiguous()
        val, wl_grad = gp2d_wirelength(prob, dp, pos_soa, n_obj, gamma)
        dens_grad = torch.zeros((n_obj, 2), dtype=torch.float64, device="cuda")
        ov = torch.zeros(4, dtype=torch.float64, device="cuda")
        ov[3:4].copy_(val)
        for layer, ctx in enumerate(layers):
            if ctx.n:
                ctx.run(p, dens_grad, ov[layer:layer + 1])
        host = ov.cpu().tolist()
        return host[3], wl_grad, dens_grad, host[:3]

    opt = NesterovOptimizer(_dev.f64(pos), project=project)
    info = GpInfo()
    lams = None
    charges = sw * sh * grids[0].db
    lay = torch.from_numpy(obj_layer).cuda()
    prev = [math.inf] * 3
    prev_raw = None
    for it in range(cfg.max_iters):
        gamma = gamma_schedule(grids[0], it, cfg.max_iters, cfg)
        val, wl_grad, dens_grad, ovfls = evaluate(opt.v, gamma)
        if lams is None:
            lams = [lambda_init(float(wl_grad[layer_idx[l]].abs().sum().item()),
                                float(dens_grad[layer_idx[l]].abs().sum().item()))
                    for l in range(3)]
        worst = max(ovfls)
        info.iterations = it + 1
        info.final_overflow = worst
        if iteration_log is not None:
            iteration_log.append((it, val, prob.n_hbt, worst))
        if worst <= cfg.stop_overflow:
            break
        lam_obj = torch.tensor(lams, dtype=torch.float64, device="cuda")[lay]
        total = wl_grad + lam_obj[:, None] * dens_grad
        pre, _ = precondition(total, 1.0, lam_obj * charges, degree_obj, is_macro_obj)
        pre_prev = None
        if prev_raw is not None:
            pre_prev, _ = precondition(prev_raw[0] + lam_obj[:, None] * prev_raw[1], 1.0,
                                       lam_obj * charges, degree_obj, is_macro_obj)
        prev_raw = (wl_grad, dens_grad)
        try:
            opt.advance(pre, step_scale=grids[0].wb, g_prev_reval=pre_prev)
        except StepUnderflow:
            info.diverged = True
            break
        for layer in range(3):
            lams[layer] *= mu_from_overflow(prev[layer], ovfls[layer], cfg)
            prev[layer] = ovfls[layer]

    final = project(opt.u).cpu().numpy()
    state.x = final[: prob.n_inst, 0].copy()
    state.y = final[: prob.n_inst, 1].copy()
    hbt_centers = {int(j): (float(final[prob.n_inst + t, 0]), float(final[prob.n_inst + t, 1]))
                   for t, j in enumerate(prob.crossing)}
    return state, info, hbt_centers


__all__ = ["Gp2dProblem", "gp2d_grid_n", "gp2d_wirelength", "run_gp2d_multi"]
