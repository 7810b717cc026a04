"""Drop-in of the ``place3d.gp`` 3D global-placement loop on the B200.

``run_gp3d`` keeps the reference signature (gp.py:359-455) but runs every
iteration on the device: one ``p3d_gp_iterate`` enqueues K1..K5 with all loop
control (lambda init, gamma/mu schedules, best-state key, stop, divergence and
step-underflow exits) in device memory, and the host replays a CUDA graph of
several iterations, polling a done flag.  The per-iteration log rows
``(it, exact WL, crossings, overflow)`` are copied back once at the end.

Host-side setup (grid choice, initial jitter, fillers, alpha) is the
reference's own numpy arithmetic so initial states are bit-identical.
"""

from __future__ import annotations

import ctypes as C
import logging
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from . import density as dn
from . import wirelength as wl
from .dist import object_slabs
from .model import PlacementState, partition_from_z, rotated_dims

log = logging.getLogger("place3d")

K_MAX_BLOCKS = 2048
# The persistent grids (K1, K4, K5) are sized for B200's 148 SMs as a constant,
# not queried: their block counts partition the ordered reductions (WL value,
# energy, norms), so a fixed count keeps the logged rows bit-identical on any
# GPU model (another SM count only over- or under-fills the one wave).
GRID_SMS = 148
K_PARTIAL_STRIDE = 8 * K_MAX_BLOCKS


class StepUnderflow(RuntimeError):
    pass


@dataclass
class GpConfig:
    """Field-for-field ``GpConfig`` (gp.py:30-50)."""

    seed: int = 1
    nz: int = 8
    grid_nx: int | None = None
    grid_ny: int | None = None
    stop_overflow: float = 0.10
    max_iters: int = 1200
    mu_min: float = 1.01
    mu_max: float = 1.05
    gamma_start_factor: float = 4.0
    gamma_end_factor: float = 0.5
    target_density: float = 1.0
    alpha: float | None = None
    alpha0: float = 3.5e-3
    cut_cost_factor: float = 5.0
    log_base: float | None = None
    flow: str = "auto"
    jitter_frac: float = 0.02
    divergence_window: int = 100
    threads: int = 1


@dataclass
class GpInfo:
    iterations: int = 0
    final_overflow: float = math.inf
    diverged: bool = False
    wirelength: float = 0.0
    hbt_count: int = 0


@dataclass
class GradientBundle:
    """Per-object gradients ([n_obj, 3]; numpy when evaluate() got numpy
    positions, else CUDA tensors) and objective parts (gp.py:62-72)."""

    wl_grad: torch.Tensor
    dens_grad: torch.Tensor
    total: torch.Tensor
    divisors: torch.Tensor
    value: float
    wl_value: float
    energy: float


# ---------------------------------------------------------------------------
# host setup (reference arithmetic, gp.py:75-175)
# ---------------------------------------------------------------------------


def choose_grid(design, cfg: GpConfig) -> dn.DensityGrid:
    """gp.py:75-87."""
    n = max(design.n_insts, 1)
    if cfg.grid_nx is not None:
        nx = cfg.grid_nx
        ny = cfg.grid_ny or cfg.grid_nx
    else:
        k = 3
        while (2 ** (k + 1)) ** 2 <= n / 4 and 2 ** (k + 1) <= 128:
            k += 1
        nx = ny = 2 ** k
    return dn.DensityGrid(design.die.width, design.die.height, nx, ny, cfg.nz)


def alpha_value(design, dz: float, cfg: GpConfig) -> float:
    """gp.py:90-107."""
    if cfg.alpha is not None:
        return cfg.alpha
    die, hbt = design.die, design.hbt
    eta = 2 * hbt.pitch / (die.row_height_top + die.row_height_bottom)
    arg = max(90 * hbt.cost * eta - 1, 1 + 1e-6)
    lg = math.log(arg) if cfg.log_base is None else math.log(arg, cfg.log_base)
    fitted = cfg.alpha0 * (die.width * eta ** 2 / dz) * lg
    floor = cfg.cut_cost_factor * hbt.cost / (dz / 2)
    return max(fitted, floor)


def select_flow(design) -> str:
    """gp.py:110-112."""
    return "2d" if design.r_ma >= 0.5 else "3d"


def init_state(design, grid, cfg: GpConfig, rng) -> PlacementState:
    """gp.py:115-126 (same rng draws)."""
    n = design.n_insts
    die = design.die
    x = np.full(n, die.width / 2) + rng.normal(0, cfg.jitter_frac * die.width, n)
    y = np.full(n, die.height / 2) + rng.normal(0, cfg.jitter_frac * die.height, n)
    z = np.full(n, grid.dz / 2) + rng.normal(0, cfg.jitter_frac * grid.dz, n)
    arr = design.arrays()
    x = np.clip(x, arr.w_bot / 2, die.width - arr.w_bot / 2)
    y = np.clip(y, arr.h_bot / 2, die.height - arr.h_bot / 2)
    z = np.clip(z, grid.dz / 4, 3 * grid.dz / 4)
    return PlacementState(x=x, y=y, z=z, rot=np.zeros(n, dtype=np.int64), dz=grid.dz)


def make_fillers(design, grid, rng) -> dn.FillerSet:
    """gp.py:129-139."""
    arr = design.arrays()
    cells = ~arr.is_macro
    if cells.any():
        hint = float(np.median(arr.w_bot[cells] * arr.h_bot[cells]))
    else:
        hint = (design.die.width / 32) ** 2
    return dn.build_fillers((design.die.width, design.die.height), grid.dz,
                            design.die.max_util_top, design.die.max_util_bottom, hint, rng)


def lambda_init(wl_norm, dens_norm, scale=1e-3):
    """gp.py:150-153 (the device loop applies the same rule)."""
    if wl_norm <= 0 or dens_norm <= 0:
        return scale
    return scale * wl_norm / dens_norm


def mu_from_overflow(prev_ovfl, cur_ovfl, cfg: GpConfig):
    """gp.py:156-168 (the device loop applies the same rule)."""
    drop = prev_ovfl - cur_ovfl
    if drop < 0:
        mu = cfg.mu_min
    elif drop >= 2e-3:
        mu = cfg.mu_min + 0.01
    elif drop >= 5e-4:
        mu = (cfg.mu_min + cfg.mu_max) / 2
    else:
        mu = cfg.mu_max
    return min(max(mu, cfg.mu_min), cfg.mu_max)


def gamma_schedule(grid, it, max_iters, cfg: GpConfig):
    """gp.py:171-175."""
    t = min(1.0, it / max(max_iters - 1, 1))
    g0 = cfg.gamma_start_factor * grid.db
    g1 = cfg.gamma_end_factor * grid.db
    return g0 * (g1 / g0) ** t


@_dev.numpy_io("gradients")
def precondition(gradients, lam, charges, pin_degrees, macro_flags):
    """Eq. 19 (gp.py:142-147) on the device: g / max(1, lam q [+ #pins])."""
    _lib.require_cuda()
    g = _dev.f64(gradients)
    shape = g.shape
    k = shape[1] if g.dim() == 2 else 0
    if k == 3:
        g = g.contiguous()
    elif k:  # [n, k] (e.g. the 2D GP's [n, 2]): padded to the kernel's 3 columns
        g = torch.cat([g, torch.zeros((g.shape[0], 3 - k), dtype=g.dtype, device=g.device)], 1)
    else:
        g = g.reshape(-1, 1).expand(-1, 3).contiguous()
    n = g.shape[0]
    q = _dev.f64(charges)
    deg = _dev.f64(pin_degrees)
    m = _dev.u8(macro_flags)
    out = torch.empty_like(g)
    div = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("p3d_precondition", int(n), _lib.ptr(g), float(lam), _lib.ptr(q), _lib.ptr(deg),
              _lib.ptr(m), _lib.ptr(out), _lib.ptr(div), _lib.stream_ptr())
    if len(shape) != 2:
        out = out[:, 0].reshape(shape)
    elif k != 3:
        out = out[:, :k].contiguous()
    return out, div


class NesterovOptimizer:
    """Accelerated descent with a clipped Barzilai-Borwein step (gp.py:178-227),
    on CUDA tensors, for callers that drive their own loop (the fused device
    loop in ``run_gp3d`` does not use this class).  The norms, max |g| and the
    two updates are device kernels (``p3d_nesterov_op``); ``project`` is the
    caller's (e.g. ``Gp3dProblem.project``)."""

    def __init__(self, x0, project=None, min_step=1e-18):
        # numpy in, numpy out (the per-op convention): a host caller's
        # `project` sees numpy arrays and `u` / `v` / `advance` return them
        self._host = not isinstance(x0, torch.Tensor)
        user = project or (lambda p: p)
        self.project = (lambda t: _dev.f64(user(_dev.host(t)))) if self._host else user
        self._u = self.project(_dev.f64(np.array(x0, dtype=float) if self._host else x0).clone())
        self._v = self._u.clone()
        self.a = 1.0
        self.step = None
        self.min_step = min_step
        self._prev_v = None
        self._prev_g = None
        self._scr = _dev.scratch(8 + 2 * 2048 + 8)
        self._out = torch.zeros(4, dtype=torch.float64, device="cuda")

    @property
    def u(self):
        return _dev.host(self._u) if self._host else self._u

    @property
    def v(self):
        return _dev.host(self._v) if self._host else self._v

    def _op(self, op, v, vp, g, ref, s=0.0, out=None):
        _lib.call("p3d_nesterov_op", int(op), int(g.numel()), _lib.ptr(v), _lib.ptr(vp),
                  _lib.ptr(g), _lib.ptr(ref), float(s), _lib.ptr(self._out if out is None else out),
                  _lib.ptr(self._scr), _lib.stream_ptr())

    def advance(self, g, step_scale=1.0, g_prev_reval=None):
        g = _dev.f64(g).contiguous()
        ref = _dev.f64(g_prev_reval).contiguous() if g_prev_reval is not None else self._prev_g
        if self.step is None or self._prev_v is None or ref is None:
            if self.step is None:
                if g.numel():
                    self._op(1, None, None, g, None)
                    gmax = float(self._out[0].item())
                else:
                    gmax = 0.0
                self.step = 1.0 if gmax == 0 else step_scale / gmax
        else:
            self._op(0, self._v, self._prev_v, g, ref)
            dv2, dg2 = self._out[:2].tolist()
            den = math.sqrt(dg2)
            if den > 0:
                new = math.sqrt(dv2) / den
                self.step = float(min(max(new, self.step / 4), self.step * 4))
        if not math.isfinite(self.step) or self.step <= self.min_step:
            raise StepUnderflow(f"step size underflow ({self.step!r})")
        self._prev_v = self._v.clone()
        self._prev_g = g.clone()
        u_new = torch.empty_like(self._v)
        self._op(2, self._v, None, g, None, -self.step, out=u_new)  # v - step * g
        u_new = self.project(u_new)
        a_new = (1 + math.sqrt(4 * self.a ** 2 + 1)) / 2
        v_new = torch.empty_like(u_new)
        self._op(2, u_new, None, u_new, self._u, (self.a - 1) / a_new, out=v_new)
        self._v = self.project(v_new)
        self._u = u_new
        self.a = a_new
        return self.u


# ---------------------------------------------------------------------------
# the device problem context
# ---------------------------------------------------------------------------


MAX_STAGED_DEG = 6  # kMaxStagedDeg in p3d_wl_fused.cu


def fused_pin_layout(net_ptr, pin_inst, off4, dup, net_key=None):
    """Host build of the fused-K1 layout.  Nets are grouped by degree and each
    degree bucket is stored transposed ([pin k][net j]) so a warp owning 32
    nets of a bucket loads pin k of all of them in one transaction.  Returns a
    dict of device-ready arrays: warp tasks, per-permuted-net (base, degree,
    stride, dup), permuted per-pin (owner, float32 offsets, owner-sorted record
    slot) and, per original pin, its permuted index.  Records are written at
    their owner-sorted slot (stable: original pin order within an owner, like
    bincount), so the owner gather streams them.  net_key (sharded halo mode):
    a secondary sort key inside each degree bucket, so nets evaluated by the
    same set of ranks share warp tasks."""
    net_ptr = np.asarray(net_ptr, dtype=np.int64)
    deg = np.diff(net_ptr)
    n_net = len(deg)
    order = _dev.stable_argsort(deg) if net_key is None else np.lexsort((net_key, deg))
    dsorted = deg[order]
    base = np.zeros(n_net, dtype=np.int64)
    stride = np.ones(n_net, dtype=np.int64)
    dest = np.empty(len(pin_inst), dtype=np.int64)
    tasks, t0s, generic = [], [], []
    pos = 0
    bounds = np.flatnonzero(np.r_[True, dsorted[1:] != dsorted[:-1], True]) if n_net else [0]
    for b0, b1 in zip(bounds[:-1], bounds[1:]):
        D = int(dsorted[b0])
        nb = int(b1 - b0)
        nets = order[b0:b1]
        j = np.arange(nb)
        base[b0:b1] = pos + j
        stride[b0:b1] = nb
        if D:
            k = np.arange(D)
            src = net_ptr[nets][:, None] + k[None, :]
            dest[src.reshape(-1)] = (pos + k[None, :] * nb + j[:, None]).reshape(-1)
        if 2 <= D <= MAX_STAGED_DEG:
            for j0 in range(0, nb, 32):
                tasks.append((pos, nb, j0, D))
                t0s.append(int(b0))
        else:
            generic.extend(range(int(b0), int(b1)))
        pos += nb * D
    off4 = np.asarray(off4, dtype=np.float64)
    off32 = off4.astype(np.float32)
    if not np.array_equal(off32.astype(np.float64), off4):
        raise ValueError("pin offsets are not exactly representable in float32")
    f_inst = np.empty_like(pin_inst)
    f_inst[dest] = pin_inst
    f_off = np.empty((len(pin_inst), 4), dtype=np.float32)
    f_off[dest] = off32
    # owner-sorted slots (stable: original pin order within an owner, like bincount)
    slot_order = _dev.stable_argsort(pin_inst)
    pin_slot = np.empty(len(pin_inst), dtype=np.int64)
    pin_slot[dest[slot_order]] = np.arange(len(pin_inst))
    return dict(tasks=np.asarray(tasks, dtype=np.int64).reshape(-1, 4),
                task_t0=np.asarray(t0s, dtype=np.int64), net_base=base, net_deg=dsorted,
                net_stride=stride, net_dup=np.asarray(dup, bool)[order], pin_inst=f_inst,
                pin_off=f_off, pin_slot=pin_slot, dest=dest,
                generic=np.asarray(generic, dtype=np.int64), order=order)


def _with_dup_nets(layout):
    """Duplicate-owner nets (exact O(|P|^2) FD path) run in the generic kernel."""
    dup_t = np.flatnonzero(layout["net_dup"])
    staged = ~np.isin(dup_t, layout["generic"])
    layout["generic"] = np.sort(np.r_[layout["generic"], dup_t[staged]]).astype(np.int64)
    return layout


class Gp3dProblem:
    """Evaluation context for one 3D GP run (gp.py:235-341), device-resident.

    Holds the p3d_gp descriptor: topology, per-object constants and all state
    buffers (HBM layout in DESIGN.md).  ``evaluate`` / ``project`` /
    ``cloud`` keep the reference semantics; ``run`` drives the fused loop."""

    def __init__(self, design, grid: dn.DensityGrid, fillers: dn.FillerSet, cfg: GpConfig, rot,
                 max_iters=None, precision=None, shard=None, min_step=1e-18):
        """precision: "fp64" (default; WA sums in float64 with numpy's
        operation order) or "fp32" (WA sums in float32 on anchor-relative
        differences, the SURVEY App. B plan; faster, ~1e-7 relative).
        min_step: the step-underflow bound of the reference's
        NesterovOptimizer (gp.py:188, default 1e-18)."""
        _lib.require_cuda()
        import os

        self.precision = precision or os.environ.get("P3D_WL_PRECISION", "fp64")
        if self.precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        self.design = design
        self.grid = grid
        self.fillers = fillers
        self.cfg = cfg
        self.rot = np.asarray(rot)
        self.arr = arr = design.arrays()
        self.topo = wl.NetTopology.from_arrays(arr)
        self.n_inst = design.n_insts
        self.n_fill = fillers.count
        self.n_obj = self.n_inst + self.n_fill
        self.alpha = alpha_value(design, grid.dz, cfg)
        self.w_top, self.h_top = rotated_dims(arr.w_top, arr.h_top, self.rot)
        self.w_bot, self.h_bot = rotated_dims(arr.w_bot, arr.h_bot, self.rot)
        self.is_macro_obj = np.r_[arr.is_macro, np.zeros(self.n_fill, bool)]
        self.degree_obj = np.r_[arr.pin_degree, np.zeros(self.n_fill)]
        self.freeze_z = np.r_[np.zeros(self.n_inst, bool), np.ones(self.n_fill, bool)]
        self.weight = np.r_[np.where(arr.is_macro, cfg.target_density, 1.0), np.ones(self.n_fill)]
        zmid = np.full(self.n_inst, grid.dz / 2)
        zc = np.clip(zmid, grid.dz / 4, 3 * grid.dz / 4)
        t = 2 * zc / grid.dz - 0.5
        up = (zc - grid.dz / 2) > 0
        wv = np.where(arr.is_macro, t * self.w_top + (1 - t) * self.w_bot,
                      np.where(up, self.w_top, self.w_bot))
        hv = np.where(arr.is_macro, t * self.h_top + (1 - t) * self.h_bot,
                      np.where(up, self.h_top, self.h_bot))
        self.movable_volume = float((wv * hv).sum() * grid.dz / 2)
        self.max_iters = int(cfg.max_iters if max_iters is None else max_iters)
        self.min_step = float(min_step)
        # shard: None (fused single-GPU loop) or (rank, world) for shard.ShardedGp3d
        # shard: (rank, world) deals K1 tasks round-robin; (rank, world, HaloPlan)
        # runs this rank's own nets (partition.py) in halo mode
        self.sharded = shard is not None
        self.shard_rank, self.shard_size = (int(shard[0]), int(shard[1])) if shard else (0, 1)
        self.plan = shard[2] if shard is not None and len(shard) > 2 else None
        self._build()

    def _halo_filter(self, L):
        """Halo mode: keep the warp tasks / generic nets holding a net that
        touches this rank's slab; mark (bit 1 of the dup byte) the nets whose
        value another rank counts."""
        mask, prim = self.plan.nets_of(self.shard_rank)
        order = L["order"]
        m_perm = mask[order]
        keep = []
        for k, (pos, nb, j0, D) in enumerate(L["tasks"]):
            t0 = int(L["task_t0"][k])
            if m_perm[t0 + j0: t0 + min(nb, j0 + 32)].any():
                keep.append(k)
        keep = np.asarray(keep, dtype=np.int64)
        L["tasks"] = L["tasks"][keep].reshape(-1, 4)
        L["task_t0"] = L["task_t0"][keep]
        L["generic"] = L["generic"][m_perm[L["generic"]]] if len(L["generic"]) else L["generic"]
        L["net_dup"] = (np.asarray(L["net_dup"], dtype=np.uint8) |
                        ((~prim[order]).astype(np.uint8) << 1))

    # -- device descriptor -------------------------------------------------
    def _build(self):
        arr, grid, cfg = self.arr, self.grid, self.cfg
        keep = self._keep = _dev.Keep()
        dt = self.topo.device(arr.net_has_dup_inst)
        self._dtopo = dt
        I, F, O = self.n_inst, self.n_fill, self.n_obj
        B = grid.n_bins
        P = arr.n_pin
        g = self.gp = _lib.Gp()
        g.n_inst, g.n_fill, g.n_obj = I, F, O
        macro_ids = np.flatnonzero(arr.is_macro).astype(np.int32)
        # this rank's objects: an instance slab of equal padded size
        # (so the pos4 slabs all-gather with equal counts) and a filler slab
        R, r = self.shard_size, self.shard_rank
        self.inst_slab, self.sh_i, self.sh_f = object_slabs(I, F, r, R)
        g.shard_rank, g.shard_size = r, (R if self.sharded else 0)
        # WL and density branches concurrently inside the iteration graph
        g.overlap = int(os.environ.get("P3D_OVERLAP", "1")) if not self.sharded else 0
        g.shard_halo = 1 if self.plan is not None else 0
        g.sh_i0, g.sh_i1 = self.sh_i
        g.sh_f0, g.sh_f1 = self.sh_f
        macro_ids = macro_ids[(macro_ids >= self.sh_i[0]) & (macro_ids < self.sh_i[1])]
        g.n_macro = len(macro_ids)
        if g.n_macro + 1 > K_MAX_BLOCKS:  # K4 runs n_macro + nblk_dens (>= 1) CTAs
            raise ValueError(f"{g.n_macro} macros exceed the per-launch CTA budget {K_MAX_BLOCKS}")
        mi = max(self.max_iters, 1)
        g.max_iters = self.max_iters
        g.divergence_window = int(cfg.divergence_window)
        # object kernels run one persistent wave of 256-thread CTAs: K5 (85
        # registers, every load hoisted) 3 per SM, K4 (64 registers) 4 per SM
        n_sm = GRID_SMS
        g.nblk_obj = max(1, min(-(-O // 256), K_MAX_BLOCKS,
                                int(os.environ.get("P3D_NBLK_OBJ", 3 * n_sm))))
        g.nblk_dens = max(1, min(-(-O // 256), K_MAX_BLOCKS - g.n_macro,
                                 int(os.environ.get("P3D_NBLK_DENS", 4 * n_sm))))
        g.nblk_net = max(1, min(-(-max(arr.n_net, 1) // 256), K_MAX_BLOCKS))
        tp = dt.struct
        g.topo = _lib.Topology(tp.n_net, tp.n_pin, I, 0, tp.net_ptr, tp.pin_inst, tp.net_dup,
                               tp.net_order, tp.pin_slot, tp.obj_slot_ptr)
        g.wl_f32 = 1 if self.precision == "fp32" else 0
        off4 = self._off4 = wl.rotated_pin_offsets(arr, self.rot) if P else np.zeros((0, 4))
        key = None
        if self.plan is not None:  # group nets by (primary rank, set of ranks touching them)
            key = self.plan.primary * (1 << R)
            for q in range(R):
                key = key + (self.plan.touches[q].astype(np.int64) << q)
        L = self.layout = _with_dup_nets(
            fused_pin_layout(arr.net_ptr, arr.pin_inst, off4, arr.net_has_dup_inst, net_key=key))
        if self.plan is not None:
            self._halo_filter(L)
        one = lambda a, dt_: a if len(a) else np.zeros(1, dt_)  # noqa: E731
        g.f_n_tasks = len(L["tasks"])
        g.f_n_generic = len(L["generic"])
        g.f_generic_nets = keep(_dev.i32(one(L["generic"], np.int64)))
        g.f_tasks = keep(_dev.i32(one(L["tasks"].reshape(-1), np.int64)))
        g.f_task_t0 = keep(_dev.i32(one(L["task_t0"], np.int64)))
        g.f_net_base = keep(_dev.i32(one(L["net_base"], np.int64)))
        g.f_net_deg = keep(_dev.i32(one(L["net_deg"], np.int64)))
        g.f_net_stride = keep(_dev.i32(one(L["net_stride"], np.int64)))
        g.f_net_dup = keep(_dev.u8(one(L["net_dup"].astype(np.uint8), np.uint8)))
        g.f_pin_inst = keep(_dev.i32(one(L["pin_inst"], np.int64)))
        g.f_pin_off = keep(_dev.dev(one(L["pin_off"].reshape(-1), np.float32), torch.float32))
        g.f_pin_slot = keep(_dev.i32(one(L["pin_slot"], np.int64)))
        # K1 runs one persistent wave of 128-thread CTAs: 4 per SM (all its
        # 124-register budget allows) alone, 3.5 per SM when it shares the GPU
        # with the density branch (measured at config 3: +0.9% over 3 per SM,
        # +1.5% over 4 per SM; 3.25 / 3.75 per SM in between)
        g.nblk_net = max(1, min(-(-g.f_n_tasks // 4), K_MAX_BLOCKS,
                                int(os.environ.get("P3D_NBLK_NET",
                                                   (7 * n_sm) // 2 if g.overlap else 4 * n_sm))))
        gs, gkeep = grid.device()
        g.grid = gs
        self._gkeep = gkeep
        self.t_pin_off = _dev.f64(self._off4 if P else np.zeros((1, 4)))
        g.pin_off = keep(self.t_pin_off)
        g.w_top = keep(_dev.f64(self.w_top if I else np.zeros(1)))
        g.h_top = keep(_dev.f64(self.h_top if I else np.zeros(1)))
        g.w_bot = keep(_dev.f64(self.w_bot if I else np.zeros(1)))
        g.h_bot = keep(_dev.f64(self.h_bot if I else np.zeros(1)))
        g.is_macro = keep(_dev.u8(arr.is_macro if I else np.zeros(1, bool)))
        g.degree = keep(_dev.f64(arr.pin_degree.astype(np.float64) if I else np.zeros(1)))
        fl = self.fillers
        g.fill_w = keep(_dev.f64(fl.w if F else np.zeros(1)))
        g.fill_h = keep(_dev.f64(fl.h if F else np.zeros(1)))
        g.fill_z = keep(_dev.f64(fl.z if F else np.zeros(1)))
        g.macro_ids = keep(_dev.i32(macro_ids if len(macro_ids) else np.zeros(1, np.int32)))
        gam = [gamma_schedule(grid, it, self.max_iters, cfg) for it in range(mi)]
        g.gamma_tab = keep(_dev.f64(np.asarray(gam, dtype=np.float64)))
        g.alpha = self.alpha
        g.target_density = cfg.target_density
        g.movable_volume = self.movable_volume
        g.stop_overflow = cfg.stop_overflow
        g.mu_min, g.mu_max = cfg.mu_min, cfg.mu_max
        g.gamma0 = cfg.gamma_start_factor * grid.db
        g.gamma1 = cfg.gamma_end_factor * grid.db
        g.min_step = self.min_step
        g.step_scale = grid.wb
        g.rho_t_fx = int(np.rint(cfg.target_density * np.ldexp(1.0, dn.FX_BITS)))
        z = lambda n: torch.zeros(max(int(n), 1), dtype=torch.float64, device="cuda")  # noqa: E731
        self.t_u, self.t_v, self.t_best = z(3 * O), z(3 * O), z(3 * O)
        self.t_vprev = z(1)  # p3d_gp.v_prev is unused (the step reduces |dv|^2 itself)
        self.t_wl, self.t_dens, self.t_pre = z(3 * O), z(3 * O), z(3 * O)
        self.t_prev_wl, self.t_prev_dens, self.t_prev_q = z(3 * O), z(3 * O), z(O)
        self.t_pin_out = z(4 * P)
        self.t_pin_out_f = torch.zeros(max(4 * P, 4), dtype=torch.float32, device="cuda")
        self.t_pin_out_fd = z(P)
        self.t_pos4 = z(4 * max(I, R * self.inst_slab))
        self.t_shard_tot = z(32)
        g.shard_tot = keep(self.t_shard_tot)
        self.t_inst_g = z(4 * max(I, R * self.inst_slab))
        self.t_rho_fx = torch.zeros(B, dtype=torch.int64, device="cuda")
        self.t_rho = z(B)
        tx, ty = -(-grid.nx // 16), -(-grid.ny // 16)  # kTile in p3d_density.cu
        nt = tx * ty
        i32z = lambda n: torch.zeros(max(int(n), 1), dtype=torch.int32, device="cuda")  # noqa: E731
        # ts_order: [O] tiles, [O] sort permutation, [1] permutation-valid flag, [1] the
        # iteration's sort decision
        self.t_ts = [i32z(O), i32z(nt), i32z(nt + 1), i32z(nt), i32z(2 * O + 2)]
        g.ts_n_tiles, g.ts_tiles_x, g.ts_tiles_y = nt, tx, ty
        # footprint reach past the centre tile, in bins (+2: centre-bin rounding)
        cell = ~arr.is_macro
        half = max([0.0] + [float(np.max(a[cell])) for a in (self.w_top, self.w_bot, self.h_top,
                                                              self.h_bot) if cell.any()] +
                   [float(np.max(a)) for a in (fl.w, fl.h) if F]) / 2
        g.ts_margin = int(np.ceil(half / min(grid.wb, grid.hb))) + 2
        for name, t in zip(("ts_tile_of", "ts_hist", "ts_start", "ts_cursor", "ts_order"), self.t_ts):
            setattr(g, name, keep(t))
        self.t_ts_rec = z(6 * O)
        g.ts_rec = keep(self.t_ts_rec)
        self.t_spec = z(6 * B)
        self.t_maps = z(4 * B)
        self.t_partials = z(_lib.load().p3d_gp_partials_doubles())
        self.t_st = torch.zeros(C.sizeof(_lib.LoopState), dtype=torch.uint8, device="cuda")
        self.t_log = z(4 * mi)
        self.t_hist = z(mi)
        for name, t in (("u", self.t_u), ("v", self.t_v), ("v_prev", self.t_vprev),
                        ("best", self.t_best), ("wl_grad", self.t_wl), ("dens_grad", self.t_dens),
                        ("pre", self.t_pre), ("prev_wl", self.t_prev_wl),
                        ("prev_dens", self.t_prev_dens), ("prev_q", self.t_prev_q),
                        ("pin_out", self.t_pin_out), ("pin_out_f", self.t_pin_out_f),
                        ("pin_out_fd", self.t_pin_out_fd), ("pos4", self.t_pos4),
                        ("inst_g", self.t_inst_g),
                        ("rho_fx", self.t_rho_fx), ("rho", self.t_rho),
                        ("spec_scratch", self.t_spec), ("maps", self.t_maps),
                        ("partials", self.t_partials), ("st", self.t_st), ("log", self.t_log),
                        ("ovfl_hist", self.t_hist)):
            setattr(g, name, keep(t))
        self._st_host = torch.empty(C.sizeof(_lib.LoopState), dtype=torch.uint8, pin_memory=True)

    # -- helpers ------------------------------------------------------------
    def _soa(self, pos):
        """[O,3] (numpy or tensor) -> [3*O] SoA device tensor."""
        p = _dev.f64(pos).reshape(self.n_obj, 3)
        return p.t().contiguous().reshape(-1)

    def _aos(self, soa):
        return soa[: 3 * self.n_obj].reshape(3, self.n_obj).t().contiguous()

    def state(self):
        """Copy of the device loop state (synchronises)."""
        self._st_host.copy_(self.t_st)
        return _lib.LoopState.from_buffer_copy(bytes(self._st_host.numpy()))

    # -- reference API ---------------------------------------------------------
    def cloud(self, pos):
        """ChargeCloud at pos [O,3] (gp.py:267-278): numpy arrays for numpy
        positions, CUDA tensors for tensors."""
        c = self._cloud(pos)
        if not isinstance(pos, torch.Tensor):
            c = dn.ChargeCloud(*(_dev.host(getattr(c, k)) for k in (
                "x", "y", "z", "w", "h", "dep", "weight", "is_macro")))
        return c

    def _cloud(self, pos):
        p = _dev.f64(pos).reshape(self.n_obj, 3)
        w, h = dn.dynamic_size(self.w_top, self.h_top, self.w_bot, self.h_bot, self.arr.is_macro,
                               p[: self.n_inst, 2], self.grid.dz)
        return dn.ChargeCloud(
            x=p[:, 0], y=p[:, 1], z=p[:, 2],
            w=torch.cat([w, _dev.f64(self.fillers.w)]), h=torch.cat([h, _dev.f64(self.fillers.h)]),
            dep=torch.full((self.n_obj,), self.grid.dz / 2, dtype=torch.float64, device="cuda"),
            weight=_dev.f64(self.weight), is_macro=self.is_macro_obj)

    def project(self, pos):
        """gp.py:280-294 on the device; [O,3] -> [O,3] tensor."""
        src = self._soa(pos)
        out = torch.empty_like(src)
        _lib.call("p3d_gp_project", _lib.byref(self.gp), _lib.ptr(src), _lib.ptr(out),
                  _lib.stream_ptr())
        out = self._aos(out)
        return out if isinstance(pos, torch.Tensor) else _dev.host(out)

    def evaluate(self, pos, lam, gamma):
        """gp.py:296-341: (GradientBundle, overflow, exact WL, crossings)."""
        self.t_v.copy_(self._soa(pos))
        self.t_rho_fx.zero_()
        _lib.call("p3d_gp_evaluate", _lib.byref(self.gp), float(lam), float(gamma),
                  _lib.stream_ptr())
        st = self.state()
        if st.nonfinite or not math.isfinite(st.value):
            raise FloatingPointError("non-finite objective or gradient")
        wl_g = self._aos(self.t_wl)
        dg = self._aos(self.t_dens)
        total = wl_g + lam * dg
        q = self._cloud(pos).charge
        _, div = precondition(total, lam, q, self.degree_obj, self.is_macro_obj)
        if not isinstance(pos, torch.Tensor):  # numpy in, numpy out
            wl_g, dg, total, div = (_dev.host(t) for t in (wl_g, dg, total, div))
        bundle = GradientBundle(wl_grad=wl_g, dens_grad=dg, total=total, divisors=div,
                                value=st.value, wl_value=st.wl_value, energy=st.energy)
        return bundle, st.ovfl, st.exact, int(st.ncross)

    def density_fx(self, pos):
        """The loop's K2 (sorted, shared-memory privatised scatter) at `pos`:
        the int64 fixed-point map [nx, ny, nz] (2^-40 per unit density)."""
        self.t_v.copy_(self._soa(pos))
        out = torch.empty(self.grid.n_bins, dtype=torch.int64, device="cuda")
        _lib.call("p3d_gp_density_fx", _lib.byref(self.gp), _lib.ptr(out), _lib.stream_ptr())
        return out.reshape(self.grid.shape)

    # -- fused loop ---------------------------------------------------------------
    def init_loop(self, pos0):
        src = self._soa(pos0)
        _lib.call("p3d_gp_init", _lib.byref(self.gp), _lib.ptr(src), _lib.stream_ptr())

    def iterate(self, n=1, steady=False):
        """n iterations; steady: without the iteration-0 initial-step kernel
        (only after the first iteration since init_loop)."""
        fn = "p3d_gp_iterate_steady" if steady else "p3d_gp_iterate"
        for _ in range(n):
            _lib.call(fn, _lib.byref(self.gp), _lib.stream_ptr())

    def capture(self, iters_per_graph=8, steady=False):
        """CUDA graph of `iters_per_graph` iterations (replayable; each
        iteration is a no-op once the device loop is done).  steady: the
        graph is for iterations after the first one (see iterate)."""
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self.iterate(iters_per_graph, steady=steady)
        torch.cuda.current_stream().wait_stream(s)
        return g

    def stepper(self, iters_per_graph=8, steady=True):
        """step(n): n iterations replaying captured graphs -- the first one
        after init_loop as p3d_gp_iterate, every later one steady, in runs of
        `iters_per_graph` per replay (the remainder one by one).  Each graph
        is launched once here (its upload) and the loop re-initialised, so
        call init_loop / step.reset() before stepping."""
        g0, g1 = self.capture(1), self.capture(1, steady=steady)
        gk = self.capture(iters_per_graph, steady=steady) if iters_per_graph > 1 else None
        for g_ in (g0, g1, gk):
            if g_ is not None:
                g_.replay()
        first = [True]

        def step(n=1):
            if n and first[0]:
                g0.replay()
                first[0] = False
                n -= 1
            if gk is not None:
                for _ in range(n // iters_per_graph):
                    gk.replay()
                n %= iters_per_graph
            for _ in range(n):
                g1.replay()

        step.reset = lambda: first.__setitem__(0, True)
        return step

    def run(self, pos0, use_graph=True, iters_per_graph=8, poll_every=4):
        """Initialise and run the loop to completion (max_iters or an exit).
        NVTX ranges mark the host phases (init, capture, each replay batch)
        for an external profiler's timeline."""
        nvtx = torch.cuda.nvtx
        with nvtx.range("p3d.gp3d.init"):
            self.init_loop(pos0)
        total = self.max_iters
        if not use_graph:
            done_calls = 0
            while done_calls < total:
                k = min(iters_per_graph, total - done_calls)
                with nvtx.range(f"p3d.gp3d.iterate[{done_calls}:{done_calls + k}]"):
                    self.iterate(k)
                done_calls += k
                if (done_calls // k) % poll_every == 0 and self.state().done:
                    break
            return self.state()
        with nvtx.range("p3d.gp3d.capture"):
            g0 = self.capture(1)  # iteration 0, with its initial-step kernel
            g = self.capture(iters_per_graph, steady=True)
        if total > 0:
            g0.replay()
        replays = -(-(total - 1) // iters_per_graph) if total > 1 else 0
        for r in range(replays):
            with nvtx.range(f"p3d.gp3d.replay[{1 + r * iters_per_graph}]"):
                g.replay()
            if (r + 1) % poll_every == 0 and self.state().done:
                break
        return self.state()

    def log_rows(self, n):
        rows = self.t_log[: 4 * n].reshape(n, 4).cpu().numpy()
        return [(int(r[0]), float(r[1]), int(r[2]), float(r[3])) for r in rows]


def run_gp3d(design, state: PlacementState, cfg: GpConfig, grid=None, iteration_log=None,
             rng=None, use_graph=True, precision=None, min_step=1e-18):
    """3D global placement (gp.py:359-455) with the whole loop on the device.
    On exit z is rounded to the die planes; returns (state, GpInfo).
    Extra keywords (not in the reference signature): use_graph, precision
    (see Gp3dProblem) and min_step (NesterovOptimizer's bound, gp.py:188)."""
    rng = rng or np.random.default_rng(cfg.seed)
    grid = dn.DensityGrid.of(grid) or choose_grid(design, cfg)
    if state.fillers is None:
        state.fillers = make_fillers(design, grid, rng)
    state.dz = grid.dz
    prob = Gp3dProblem(design, grid, state.fillers, cfg, state.rot, precision=precision,
                       min_step=min_step)
    n = prob.n_inst
    pos0 = np.zeros((prob.n_obj, 3))
    pos0[:n] = np.c_[state.x, state.y, state.z]
    pos0[n:] = np.c_[state.fillers.x, state.fillers.y, state.fillers.z]
    st = prob.run(pos0, use_graph=use_graph)
    info = GpInfo(iterations=st.iterations, final_overflow=st.final_overflow,
                  diverged=bool(st.diverged), wirelength=st.wirelength, hbt_count=st.hbt_count)
    if st.diverged:
        log.warning("gp3d: loop exited early (non-finite, divergence or step underflow); "
                    "returning best state")
    if iteration_log is not None:
        iteration_log.extend(prob.log_rows(st.iterations))
    src = prob.t_u if info.final_overflow <= cfg.stop_overflow else prob.t_best
    fin = torch.empty_like(src)
    _lib.call("p3d_gp_project", _lib.byref(prob.gp), _lib.ptr(src), _lib.ptr(fin),
              _lib.stream_ptr())
    final = prob._aos(fin).cpu().numpy()
    state.x = final[:n, 0].copy()
    state.y = final[:n, 1].copy()
    state.z = final[:n, 2].copy()
    state.fillers.x = final[n:, 0].copy()
    state.fillers.y = final[n:, 1].copy()
    delta = partition_from_z(state.z, grid.dz)
    state.z = np.where(delta == 1, 3 * grid.dz / 4, grid.dz / 4)
    return state, info


def __getattr__(name):
    """gp.Gp2dProblem / gp.run_gp2d_multi (gp.py:463-690) live in gp2d.py
    (imported lazily: gp2d builds on this module)."""
    if name in ("Gp2dProblem", "run_gp2d_multi"):
        from . import gp2d

        return getattr(gp2d, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


__all__ = [
    "GpConfig", "GpInfo", "GradientBundle", "StepUnderflow", "choose_grid", "alpha_value",
    "select_flow", "init_state", "make_fillers", "precondition", "lambda_init",
    "mu_from_overflow", "gamma_schedule", "NesterovOptimizer", "Gp3dProblem", "run_gp3d",
]
