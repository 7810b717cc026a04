"""Drop-in of ``place3d.density`` on the B200 (K2/K3/K4 kernels of libp3d.so).

Same names and argument meaning as ``pkg/src/place3d/density.py``; maps and
per-object arrays come back as CUDA float64 tensors.  The density map is
accumulated in int64 fixed point (2^-40 per unit density) — exact and
order-independent — and converted to float64 once.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .model import partition_from_z

FX_BITS = 40


def _pass_twiddles(n):
    """Per-pass twiddles of the fast path's in-place mixed-radix DIF FFT
    (p3d_spectral_fast.cu): for each radix-8 pass with span > 1, W_{8 span}^{q j}
    for q = 1..7, j < span, laid out [pass][q-1][j] as (cos, sin) pairs.  Empty
    unless n is a power of two in [8, 1024]."""
    L = int(n).bit_length() - 1
    if n < 8 or n > 1024 or (1 << L) != n:
        return np.zeros(0)
    out = []
    for s in range(L // 3):
        ls = L - 3 * (s + 1)
        if ls <= 0:
            continue
        span = 1 << ls
        q, j = np.meshgrid(np.arange(1, 8), np.arange(span), indexing="ij")
        ang = -2 * np.pi * (q * j) / (8 * span)
        out.append(np.stack([np.cos(ang), np.sin(ang)], -1).reshape(-1))
    return np.concatenate(out) if out else np.zeros(0)


def _tables(n, d):
    """Per-axis device tables: omega, FFT twiddles (the half table e^{-2 pi i j/n},
    j < n/2, followed by the fast path's per-pass table), DCT phase factors."""
    omega = np.pi * np.arange(n) / d
    j = np.arange(max(n // 2, 1))
    tw = np.empty((len(j), 2))
    tw[:, 0] = np.cos(2 * np.pi * j / n)
    tw[:, 1] = -np.sin(2 * np.pi * j / n)
    tw = np.concatenate([tw.reshape(-1), _pass_twiddles(n)])
    k = np.arange(n)
    ph = np.empty((n, 2))
    ph[:, 0] = np.cos(np.pi * k / (2 * n))
    ph[:, 1] = np.sin(np.pi * k / (2 * n))
    return omega, tw, ph.reshape(-1)


class DensityGrid:
    """Uniform nx x ny x nz bins over [0,dx] x [0,dy] x [0,dz] (density.py:26-55)."""

    def __init__(self, dx, dy, nx, ny, nz):
        self.dx = float(dx)
        self.dy = float(dy)
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.wb = self.dx / self.nx
        self.hb = self.dy / self.ny
        self.db = (self.wb + self.hb) / 2
        self.dz = self.nz * self.db
        self.shape = (self.nx, self.ny, self.nz)
        self.bin_vol = self.wb * self.hb * self.db
        wx = np.pi * np.arange(self.nx) / self.dx
        wy = np.pi * np.arange(self.ny) / self.dy
        wz = np.pi * np.arange(self.nz) / self.dz
        self.omega = (wx, wy, wz)
        lam = wx[:, None, None] ** 2 + wy[None, :, None] ** 2 + wz[None, None, :] ** 2
        inv = np.zeros_like(lam)
        inv[lam > 0] = 1.0 / lam[lam > 0]
        self.inv_lam = inv
        self.fx_scale = np.ldexp(1.0, FX_BITS) / self.bin_vol
        self._dev = None

    @property
    def extents(self):
        return self.wb, self.hb, self.db

    @property
    def n_bins(self):
        return self.nx * self.ny * self.nz

    @classmethod
    def of(cls, grid):
        """This class for any grid with the reference's (dx, dy, nx, ny, nz)
        (e.g. place3d.density.DensityGrid, as flow.run_flow passes it)."""
        if grid is None or isinstance(grid, cls):
            return grid
        return cls(grid.dx, grid.dy, grid.nx, grid.ny, grid.nz)

    def device(self):
        """ctypes ``p3d_grid`` + the device tables it points at (cached)."""
        if self._dev is not None:
            return self._dev
        keep = _dev.Keep()
        g = _lib.Grid()
        g.nx, g.ny, g.nz = self.nx, self.ny, self.nz
        g.dx, g.dy, g.dz = self.dx, self.dy, self.dz
        g.wb, g.hb, g.db, g.bin_vol = self.wb, self.hb, self.db, self.bin_vol
        g.fx_scale = self.fx_scale
        for a, (n, d) in enumerate(((self.nx, self.dx), (self.ny, self.dy), (self.nz, self.dz))):
            om, tw, ph = _tables(n, d)
            g.omega[a] = keep(_dev.f64(om)).value
            g.twiddle[a] = keep(_dev.f64(tw)).value
            g.phase[a] = keep(_dev.f64(ph)).value
        self._dev = (g, keep)
        return self._dev


@dataclass
class ChargeCloud:
    """Struct-of-arrays charges (density.py:58-83); numpy or CUDA tensors."""

    x: object
    y: object
    z: object
    w: object
    h: object
    dep: object
    weight: object
    is_macro: object

    @property
    def volume(self):
        return self.w * self.h * self.dep

    @property
    def charge(self):
        return self.weight * self.volume

    def subset(self, mask):
        return ChargeCloud(self.x[mask], self.y[mask], self.z[mask], self.w[mask], self.h[mask],
                           self.dep[mask], self.weight[mask], self.is_macro[mask])


class _DevCloud:
    def __init__(self, cloud: ChargeCloud, macro_override=None):
        keep = self.keep = _dev.Keep()
        self.t = {k: _dev.f64(getattr(cloud, k)) for k in ("x", "y", "z", "w", "h", "dep", "weight")}
        m = cloud.is_macro if macro_override is None else macro_override
        m = m.detach().cpu().numpy() if isinstance(m, torch.Tensor) else np.asarray(m)
        m = np.broadcast_to(np.asarray(m, dtype=bool), (self.t["x"].numel(),))
        self.is_macro = _dev.u8(m)
        ids = np.flatnonzero(m).astype(np.int32)
        self.macro_ids = _dev.i32(ids if len(ids) else np.zeros(1, np.int32))
        c = _lib.Cloud()
        c.n = self.t["x"].numel()
        c.n_macro = len(ids)
        for k, v in self.t.items():
            setattr(c, k, keep(v))
        c.is_macro = keep(self.is_macro)
        c.macro_ids = keep(self.macro_ids)
        self.struct = c
        self.n = c.n


@dataclass
class FillerSet:
    """Dummy charges enforcing per-die utilisation (density.py:86-104)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    die: np.ndarray
    w: np.ndarray
    h: np.ndarray
    dep: float

    @property
    def count(self):
        return len(self.x)

    def total_volume(self, die):
        m = self.die == die
        return float((self.w[m] * self.h[m]).sum() * self.dep)


def build_fillers(die_area_wh, dz, u_top, u_bot, cell_area_hint, rng):
    """Fillers near the typical cell footprint, exact per-die volume
    (density.py:107-131; host setup, rng draws in the reference order)."""
    dx, dy = die_area_wh
    parts = []
    for die, u in ((0, u_bot), (1, u_top)):
        area = dx * dy * (1.0 - u)
        if area <= 0:
            continue
        side_hint = max(np.sqrt(cell_area_hint), 1e-9)
        count = int(np.clip(round(area / side_hint ** 2), 1, 20000))
        side = np.sqrt(area / count)
        xs = rng.uniform(side / 2, dx - side / 2, count)
        ys = rng.uniform(side / 2, dy - side / 2, count)
        parts.append((xs, ys, np.full(count, dz / 4 if die == 0 else 3 * dz / 4),
                      np.full(count, die, dtype=np.int8), np.full(count, side),
                      np.full(count, side)))
    if not parts:
        e = np.zeros(0)
        return FillerSet(e, e, e, np.zeros(0, np.int8), e, e, dz / 2)
    cols = [np.concatenate([p[i] for p in parts]) for i in range(6)]
    return FillerSet(*cols, dz / 2)


@_dev.numpy_io("z")
def dynamic_size(w_top, h_top, w_bot, h_bot, is_macro, z, dz):
    """Footprint vs depth (density.py:134-147, Eqs. 6-7): cells switch at the
    midplane, macros blend linearly over z in [dz/4, 3dz/4] (p3d_dynamic_size)."""
    _lib.require_cuda()
    zt = _dev.f64(z).reshape(-1)
    n = zt.numel()
    wt, ht, wb, hb = (_dev.f64(np.broadcast_to(a, (n,)) if not isinstance(a, torch.Tensor)
                               else a).reshape(-1) for a in (w_top, h_top, w_bot, h_bot))
    m = _dev.u8(np.broadcast_to(np.asarray(is_macro, dtype=bool), (n,))
                if not isinstance(is_macro, torch.Tensor) else is_macro)
    w, h = torch.empty_like(zt), torch.empty_like(zt)
    _lib.call("p3d_dynamic_size", int(n), _lib.ptr(wt), _lib.ptr(ht), _lib.ptr(wb), _lib.ptr(hb),
              _lib.ptr(m), _lib.ptr(zt), float(dz), _lib.ptr(w), _lib.ptr(h), _lib.stream_ptr())
    return w, h


# ---------------------------------------------------------------------------
# accumulation (K2)
# ---------------------------------------------------------------------------


def accumulate_density_fx(grid: DensityGrid, cloud: ChargeCloud, macro_override=None):
    """int64 map [nx, ny, nz] in units of 2^-40 (the exact device map)."""
    _lib.require_cuda()
    g, _ = grid.device()
    dc = _DevCloud(cloud, macro_override)
    rho = torch.zeros(grid.shape, dtype=torch.int64, device="cuda")
    if dc.n:
        _lib.call("p3d_accumulate_density", _lib.byref(g), _lib.byref(dc.struct), _lib.ptr(rho),
                  _lib.stream_ptr())
    return rho


def fx_to_density(rho_fx):
    out = torch.empty(rho_fx.shape, dtype=torch.float64, device="cuda")
    _lib.call("p3d_fx_to_density", int(rho_fx.numel()), _lib.ptr(rho_fx), _lib.ptr(out),
              _lib.stream_ptr())
    return out


@_dev.numpy_io("cloud")
def accumulate_density(grid, cloud):
    """Density map (density.py:301-311): cells/fillers thread-per-object,
    macros one CTA each over their footprint tile."""
    return fx_to_density(accumulate_density_fx(grid, cloud))


@_dev.numpy_io("cloud")
def direct_density(grid, cloud):
    """Per-object traversal of every given charge (density.py:199-204)."""
    return fx_to_density(accumulate_density_fx(grid, cloud, macro_override=False))


@_dev.numpy_io("cloud")
def macro_prefix_density(grid, cloud):
    """Macro map (density.py:291-298); on the device every charge takes the
    per-macro tile path, which equals the corner-stamp prefix sum exactly in
    real arithmetic (Theorem 1)."""
    return fx_to_density(accumulate_density_fx(grid, cloud, macro_override=True))


@_dev.numpy_io("a")
def prefix_sum_3d(a):
    """Inclusive prefix sum along x, y, z (density.py:207-209; p3d_prefix_sum_3d)."""
    return _scan3(a, 0)


@_dev.numpy_io("a")
def suffix_sum_3d(a):
    """Adjoint of prefix_sum_3d (density.py:212-217)."""
    return _scan3(a, 1)


def _scan3(a, reverse):
    _lib.require_cuda()
    t = _dev.f64(a).clone()
    nx, ny, nz = t.shape
    _lib.call("p3d_prefix_sum_3d", int(nx), int(ny), int(nz), int(reverse), _lib.ptr(t),
              _lib.stream_ptr())
    return t


# ---------------------------------------------------------------------------
# spectral solve (K3)
# ---------------------------------------------------------------------------


def _spectral(grid, rho=None, coef=None, want_coef=False):
    _lib.require_cuda()
    g, _ = grid.device()
    B = grid.n_bins
    maps = torch.empty((B, 4), dtype=torch.float64, device="cuda")
    scr = torch.empty(6 * B, dtype=torch.float64, device="cuda")
    out_coef = None
    if coef is None:
        r = _dev.f64(rho)
        out_coef = torch.empty(grid.shape, dtype=torch.float64, device="cuda") if want_coef else None
        _lib.call("p3d_spectral", _lib.byref(g), _lib.ptr(r), _lib.ptr(out_coef), _lib.ptr(maps),
                  _lib.ptr(scr), _lib.stream_ptr())
    else:
        c = _dev.f64(coef)
        _lib.call("p3d_spectral_from_coef", _lib.byref(g), _lib.ptr(c), _lib.ptr(maps),
                  _lib.ptr(scr), _lib.stream_ptr())
    return maps, out_coef


@_dev.numpy_io("rho")
def solve_potential(rho, grid):
    """Neumann Poisson solve by cosine transforms, DC dropped
    (density.py:319-328).  Returns (phi, scipy-normalised DCT-II coef)."""
    maps, coef = _spectral(grid, rho=rho, want_coef=True)
    return maps[:, 0].reshape(grid.shape).contiguous(), coef


@_dev.numpy_io("coef")
def electric_field(coef, grid):
    """E = -grad(phi) evaluated spectrally (density.py:357-368)."""
    maps, _ = _spectral(grid, coef=coef)
    return tuple(maps[:, k].reshape(grid.shape).contiguous() for k in (1, 2, 3))


@_dev.numpy_io("rho")
def potential_and_field(rho, grid):
    """Both at once as the interleaved [B][4] (phi, Ex, Ey, Ez) map the
    density gather reads (what the fused loop uses)."""
    maps, _ = _spectral(grid, rho=rho)
    return maps


# ---------------------------------------------------------------------------
# energy / force / overflow (K4)
# ---------------------------------------------------------------------------


def _interleave(grid, phi=None, ex=None, ey=None, ez=None):
    B = grid.n_bins
    m = torch.zeros((B, 4), dtype=torch.float64, device="cuda")
    for k, a in enumerate((phi, ex, ey, ez)):
        if a is not None:
            m[:, k] = _dev.f64(a).reshape(-1)
    return m


def _gather(grid, cloud, maps, freeze_z=None):
    _lib.require_cuda()
    g, _ = grid.device()
    dc = _DevCloud(cloud)
    force = torch.zeros((dc.n, 3), dtype=torch.float64, device="cuda")
    energy = torch.zeros(1, dtype=torch.float64, device="cuda")
    fr = None if freeze_z is None else _dev.u8(freeze_z)
    scr = _dev.scratch(8 + dc.struct.n_macro + 1024 + 8)
    if dc.n:
        _lib.call("p3d_density_gather", _lib.byref(g), _lib.byref(dc.struct), _lib.ptr(maps),
                  _lib.ptr(fr), _lib.ptr(energy), _lib.ptr(force), _lib.ptr(scr),
                  _lib.stream_ptr())
    return float(energy.item()), force


def density_energy(grid, cloud, phi):
    """U = sum q * overlap-weighted mean phi (density.py:568-579)."""
    return _gather(grid, cloud, _interleave(grid, phi=phi))[0]


@_dev.numpy_io("ex")
def density_force(grid, cloud, ex, ey, ez, freeze_z=None):
    """-2 q * overlap-weighted mean E (density.py:582-609)."""
    return _gather(grid, cloud, _interleave(grid, ex=ex, ey=ey, ez=ez), freeze_z)[1]


@_dev.numpy_io("phi")
def density_energy_and_gradient(grid, cloud, phi, ex=None, ey=None, ez=None, freeze_z=None):
    """Energy U = sum q * phibar and its EXACT gradient (density.py:533-565):
    cells through the two face columns of each axis, macros through their
    differentiated corner stamps against the suffix-summed potential.  The
    field maps are accepted for interface symmetry and unused, as in the
    reference."""
    _lib.require_cuda()
    g, _ = grid.device()
    dc = _DevCloud(cloud)
    grad = torch.zeros((dc.n, 3), dtype=torch.float64, device="cuda")
    energy = torch.zeros(1, dtype=torch.float64, device="cuda")
    fr = None if freeze_z is None else _dev.u8(freeze_z)
    scr = _dev.scratch(grid.n_bins + 8 + 1024)
    phi_d = _dev.f64(phi).reshape(-1).contiguous()  # alive until the kernel ran
    if dc.n:
        _lib.call("p3d_density_energy_gradient", _lib.byref(g), _lib.byref(dc.struct),
                  _lib.ptr(phi_d), _lib.ptr(fr),
                  _lib.ptr(energy), _lib.ptr(grad), _lib.ptr(scr), _lib.stream_ptr())
    return float(energy.item()), grad


def density_energy_and_force(grid, cloud, maps, freeze_z=None):
    """Energy and force from one interleaved map in one gather pass."""
    return _gather(grid, cloud, maps, freeze_z)


def overflow(rho, grid, rho_t, movable_volume):
    """Fraction of movable volume above the target density (density.py:612-617;
    p3d_overflow)."""
    if movable_volume <= 0:
        return 0.0
    _lib.require_cuda()
    r = _dev.f64(rho).reshape(-1)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    scr = _dev.scratch(8 + 1024 + 8)
    _lib.call("p3d_overflow", int(r.numel()), _lib.ptr(r), float(rho_t), float(grid.bin_vol),
              float(movable_volume), _lib.ptr(out), _lib.ptr(scr), _lib.stream_ptr())
    return float(out.item())


def macro_overflow(grid, cloud, rho_t):
    """Overflow of the macro-only density map (density.py:620-627): the macros'
    per-macro tile map (K2) and the overflow kernel."""
    m = np.asarray(cloud.is_macro.cpu() if isinstance(cloud.is_macro, torch.Tensor)
                   else cloud.is_macro, dtype=bool)
    if not m.any():
        return 0.0
    idx = np.flatnonzero(m)
    sel = (lambda v: v[torch.from_numpy(idx).to(v.device)]) if isinstance(cloud.x, torch.Tensor) \
        else (lambda v: np.asarray(v)[idx])
    big = ChargeCloud(*(sel(getattr(cloud, k)) for k in ("x", "y", "z", "w", "h", "dep",
                                                          "weight")), is_macro=np.ones(len(idx), bool))
    vol = float(_dev.f64(big.w * big.h * big.dep).sum().item()) if isinstance(big.w, torch.Tensor) \
        else float(np.sum(big.w * big.h * big.dep))
    rho = macro_prefix_density(grid, big)
    return overflow(rho, grid, rho_t, vol)


def corner_map(corner, grid):
    """Sparse stamp of one cuboid corner (density.py:220-240): host helper of
    the corner-stamp formulation (the device path stamps whole macro tiles)."""
    xh, yh, zh = corner[0] / grid.wb, corner[1] / grid.hb, corner[2] / grid.db
    idx = []
    for base, n in ((xh, grid.nx), (yh, grid.ny), (zh, grid.nz)):
        i0 = int(np.floor(base))
        ax = [(i0, 1.0 - (base - i0)), (i0 + 1, base - i0)]
        idx.append([(i, v) for i, v in ax if 0 <= i < n and v != 0.0])
    out_idx, out_val = [], []
    for i, vi in idx[0]:
        for j, vj in idx[1]:
            for k, vk in idx[2]:
                out_idx.append((i, j, k))
                out_val.append(vi * vj * vk)
    return out_idx, out_val


def dump_fields(path_prefix, grid, named_maps):
    """Debug dump, one flat float64 file per map with a text header line
    (density.py:630-640; the reference's format)."""
    paths = []
    for name, m in named_maps.items():
        path = f"{path_prefix}{name}.bin"
        arr = np.ascontiguousarray(_dev.host(m), dtype=np.float64)
        with open(path, "wb") as fh:
            fh.write(f"{name} float64 {grid.nx} {grid.ny} {grid.nz}\n".encode())
            fh.write(arr.tobytes())
        paths.append(path)
    return paths


def load_field(path):
    """density.py:643-647."""
    with open(path, "rb") as fh:
        header = fh.readline().decode().split()
        data = np.frombuffer(fh.read(), dtype=header[1])
    return header[0], data.reshape([int(t) for t in header[2:]])


def overflow_fx(rho_fx, grid, rho_t, movable_volume):
    """Overflow straight from the int64 map (exact integer excess)."""
    g, _ = grid.device()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    scr = _dev.scratch(8 + 1024 + 8)
    _lib.call("p3d_overflow_fx", _lib.byref(g), _lib.ptr(rho_fx.contiguous()), float(rho_t),
              float(movable_volume), _lib.ptr(out), _lib.ptr(scr), _lib.stream_ptr())
    return float(out.item())


__all__ = [
    "DensityGrid", "ChargeCloud", "FillerSet", "build_fillers", "dynamic_size",
    "accumulate_density", "accumulate_density_fx", "fx_to_density", "direct_density",
    "macro_prefix_density", "prefix_sum_3d", "suffix_sum_3d", "solve_potential",
    "electric_field", "potential_and_field", "density_energy", "density_force",
    "density_energy_and_gradient",
    "density_energy_and_force", "overflow", "overflow_fx", "partition_from_z",
    "macro_overflow", "corner_map", "dump_fields", "load_field",
]
