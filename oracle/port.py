"""CPU restatement of the reference GP inner loop (TEST INFRASTRUCTURE ONLY).

Every routine below restates one reference routine of ``place3d``
(``/root/reference/pkg/src/place3d``; cited as file:line) in numpy/scipy, with
the same floating-point operation order wherever the result is compared
bit-for-bit (net boxes, finite-difference depth gradient, direct density
terms).  Third-party arithmetic is the same as the reference's: numpy ufuncs
and ``scipy.fft`` (pocketfft) DCT/DST, both unpinned in the reference
(``pkg/pyproject.toml:9-12``); the image ships numpy 2.3.5 / scipy 1.18.1.

Pinned by ``tests/test_oracle.py`` against fixtures the reference itself
produced (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field

import numpy as np
from scipy import fft as sfft

_INF = np.inf


# ==========================================================================
# grid (density.py:26-55)
# ==========================================================================


class Grid:
    def __init__(self, dx, dy, nx, ny, nz):
        self.dx, self.dy = float(dx), float(dy)
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.wb = self.dx / self.nx
        self.hb = self.dy / self.ny
        self.db = (self.wb + self.hb) / 2
        self.dz = self.nz * self.db
        self.shape = (self.nx, self.ny, self.nz)
        self.bin_vol = self.wb * self.hb * self.db
        om = [np.pi * np.arange(n) / d for n, d in
              ((self.nx, self.dx), (self.ny, self.dy), (self.nz, self.dz))]
        self.omega = tuple(om)
        lam = om[0][:, None, None] ** 2 + om[1][None, :, None] ** 2 + om[2][None, None, :] ** 2
        inv = np.zeros_like(lam)
        pos = lam > 0
        inv[pos] = 1.0 / lam[pos]
        self.inv_lam = inv


# ==========================================================================
# pins and boxes (wirelength.py:101-170, 308-322; model.py:278-318)
# ==========================================================================


def below_or_on_mid(z, dz):
    return np.asarray(z) - dz / 2 > 0  # partition_from_z, model.py:316-318 (True = top)


def turn_offsets(ox, oy, q):
    """model.py:278-289: q quarter turns counter-clockwise."""
    q = np.asarray(q) % 4
    rx = np.choose(q, [ox, -oy, -ox, oy])
    ry = np.choose(q, [oy, ox, -oy, -ox])
    return rx, ry


def pins_at(arr, x, y, z, rot, dz):
    """wirelength.py:308-322 — offsets picked by the owner's current die."""
    top = below_or_on_mid(z, dz)[arr.pin_inst]
    q = np.asarray(rot)[arr.pin_inst]
    txo, tyo = turn_offsets(arr.ox_top, arr.oy_top, q)
    bxo, byo = turn_offsets(arr.ox_bot, arr.oy_bot, q)
    px = np.asarray(x)[arr.pin_inst] + np.where(top, txo, bxo)
    py = np.asarray(y)[arr.pin_inst] + np.where(top, tyo, byo)
    pz = np.asarray(z)[arr.pin_inst]
    return px, py, pz, top


class Boxes:
    """Per (net, die) first/second extrema with multiplicity
    (wirelength.py:101-142), computed with scatter-max instead of a sort."""

    def __init__(self, pin_net, n_net, c, top):
        c = np.asarray(c, dtype=np.float64)
        seg = pin_net * 2 + np.asarray(top, dtype=np.int64)
        ns = 2 * n_net
        self.cnt = np.bincount(seg, minlength=ns).reshape(n_net, 2)
        hi1 = np.full(ns, -_INF)
        lo1 = np.full(ns, _INF)
        np.maximum.at(hi1, seg, c)
        np.minimum.at(lo1, seg, c)
        at_hi = c == hi1[seg]
        at_lo = c == lo1[seg]
        n_hi = np.bincount(seg[at_hi], minlength=ns)
        n_lo = np.bincount(seg[at_lo], minlength=ns)
        hi_rest = np.full(ns, -_INF)
        lo_rest = np.full(ns, _INF)
        np.maximum.at(hi_rest, seg[~at_hi], c[~at_hi])
        np.minimum.at(lo_rest, seg[~at_lo], c[~at_lo])
        self.max1 = hi1.reshape(n_net, 2)
        self.min1 = lo1.reshape(n_net, 2)
        self.max2 = np.where(n_hi >= 2, hi1, hi_rest).reshape(n_net, 2)
        self.min2 = np.where(n_lo >= 2, lo1, lo_rest).reshape(n_net, 2)
        self.full_min = np.minimum(self.min1[:, 0], self.min1[:, 1])
        self.full_max = np.maximum(self.max1[:, 0], self.max1[:, 1])

    def spans(self):
        top = np.where(self.cnt[:, 1] > 0, self.max1[:, 1] - self.min1[:, 1], 0.0)
        bot = np.where(self.cnt[:, 0] > 0, self.max1[:, 0] - self.min1[:, 0], 0.0)
        full = np.where(self.cnt.sum(axis=1) > 0, self.full_max - self.full_min, 0.0)
        return top, bot, full

    def bistratal(self):
        t, b, f = self.spans()
        return np.maximum(f, t + b)  # wirelength.py:167-170


# ==========================================================================
# weighted-average smoothing (wirelength.py:58-98, 173-198)
# ==========================================================================


def wa_one(v, gamma):
    """wirelength.py:58-73 for one coordinate set."""
    v = np.asarray(v, dtype=float)
    if v.size == 0:
        return 0.0, np.zeros(0)
    a = np.exp((v - v.max()) / gamma)
    b = np.exp((v.min() - v) / gamma)
    p = (v * a).sum() / a.sum()
    m = (v * b).sum() / b.sum()
    g = a / a.sum() * (1 + (v - p) / gamma) - b / b.sum() * (1 - (v - m) / gamma)
    return float(p - m), g


def wa_segments(seg, nseg, v, gamma):
    """wirelength.py:76-98: WA span per segment and its per-pin gradient."""
    hi = np.full(nseg, -_INF)
    lo = np.full(nseg, _INF)
    np.maximum.at(hi, seg, v)
    np.minimum.at(lo, seg, v)
    a = np.exp((v - hi[seg]) / gamma)
    b = np.exp((lo[seg] - v) / gamma)
    sa = np.bincount(seg, weights=a, minlength=nseg)
    sva = np.bincount(seg, weights=v * a, minlength=nseg)
    sb = np.bincount(seg, weights=b, minlength=nseg)
    svb = np.bincount(seg, weights=v * b, minlength=nseg)
    live = sa > 0
    p = np.where(live, sva / np.where(live, sa, 1), 0.0)
    m = np.where(live, svb / np.where(live, sb, 1), 0.0)
    g = a / sa[seg] * (1 + (v - p[seg]) / gamma) - b / sb[seg] * (1 - (v - m[seg]) / gamma)
    return np.where(live, p - m, 0.0), g


def planar_wl(pin_net, n_net, px, py, top, gamma, bx=None, by=None):
    """wirelength.py:173-192: branch per net/axis from unsmoothed spans."""
    dseg = pin_net * 2 + np.asarray(top, dtype=np.int64)
    val = 0.0
    out = []
    for c, bb in ((px, bx), (py, by)):
        bb = bb or Boxes(pin_net, n_net, c, top)
        t, b, f = bb.spans()
        split = t + b > f
        vf, gf = wa_segments(pin_net, n_net, c, gamma)
        vd, gd = wa_segments(dseg, 2 * n_net, c, gamma)
        val += float(np.where(split, vd[0::2] + vd[1::2], vf).sum())
        out.append(np.where(split[pin_net], gd, gf))
    return val, out[0], out[1]


def zcut(pin_net, n_net, pz, gamma):
    """wirelength.py:195-198."""
    v, g = wa_segments(pin_net, n_net, np.asarray(pz, float), gamma)
    return float(v.sum()), g


# ==========================================================================
# finite-difference depth gradient (wirelength.py:201-305)
# ==========================================================================


def _ext(vals):
    return float(vals.max() - vals.min()) if vals.size else 0.0


def bistratal_one(c, top):
    """wirelength.py:145-150."""
    c = np.asarray(c, float)
    top = np.asarray(top, bool)
    return max(_ext(c), _ext(c[top]) + _ext(c[~top]))


def flip_delta(pin_net, bb: Boxes, c, top):
    """wirelength.py:227-248: extent change when one pin alone changes die."""
    d = np.asarray(top, dtype=np.int64)
    o = 1 - d
    n = pin_net
    hi1, hi2 = bb.max1[n, d], bb.max2[n, d]
    lo1, lo2 = bb.min1[n, d], bb.min2[n, d]
    with np.errstate(invalid="ignore"):
        same = np.where(bb.cnt[n, d] <= 1, 0.0,
                        np.where(c == hi1, hi2, hi1) - np.where(c == lo1, lo2, lo1))
    other = np.maximum(bb.max1[n, o], c) - np.minimum(bb.min1[n, o], c)
    t, b, f = bb.spans()
    now = np.maximum(f, t + b)
    return np.maximum(f[n], same + other) - now[n]


def fd_depth_grad(net_ptr, pin_net, pin_inst, n_obj, px, py, top, dz, dup=None,
                  bx=None, by=None):
    """wirelength.py:251-293 (clean nets O(1)/pin, duplicate-owner nets exact)."""
    top = np.asarray(top, bool)
    n_net = len(net_ptr) - 1
    if dup is None:
        dup = np.zeros(n_net, bool)
        if len(pin_inst) > 1:
            k = np.lexsort((pin_inst, pin_net))
            rep = (np.diff(pin_net[k]) == 0) & (np.diff(pin_inst[k]) == 0)
            dup[pin_net[k[1:][rep]]] = True
    g = np.zeros(n_obj)
    clean = ~dup[pin_net]
    if clean.any():
        dw = np.zeros(len(pin_net))
        for c, bb in ((px, bx), (py, by)):
            bb = bb or Boxes(pin_net, n_net, c, top)
            dw += flip_delta(pin_net, bb, np.asarray(c, float), top)
        signed = np.where(top, -dw, dw) * (4.0 / dz)
        g += np.bincount(pin_inst[clean], weights=signed[clean], minlength=n_obj)
    scale = 4.0 / dz
    for j in np.flatnonzero(dup):
        s = slice(net_ptr[j], net_ptr[j + 1])
        xs, ys, own, tp = px[s], py[s], pin_inst[s], top[s]
        for w in np.unique(own):
            m = own == w
            up = bistratal_one(xs, np.where(m, True, tp)) + bistratal_one(ys, np.where(m, True, tp))
            dn = bistratal_one(xs, np.where(m, False, tp)) + bistratal_one(ys, np.where(m, False, tp))
            g[w] += scale * (up - dn)
    return g


def fd_depth_grad_naive(net_ptr, pin_inst, n_obj, px, py, top, dz):
    """wirelength.py:205-224: per owner, re-evaluate with the owner forced up / down."""
    g = np.zeros(n_obj)
    for j in range(len(net_ptr) - 1):
        s = slice(net_ptr[j], net_ptr[j + 1])
        xs, ys, own, tp = px[s], py[s], pin_inst[s], top[s]
        for w in np.unique(own):
            m = own == w
            up = bistratal_one(xs, np.where(m, True, tp)) + bistratal_one(ys, np.where(m, True, tp))
            dn = bistratal_one(xs, np.where(m, False, tp)) + bistratal_one(ys, np.where(m, False, tp))
            g[w] += (4.0 / dz) * (up - dn)
    return g


def normalize_depth(gx, gy, gzb, gzh, alpha):
    """wirelength.py:296-305 (Eq. 17)."""
    nz = np.abs(gzb).sum()
    if nz == 0:
        base = np.zeros_like(gzb)
    else:
        base = (np.abs(gx).sum() + np.abs(gy).sum()) / (2 * nz) * gzb
    return base + alpha * np.asarray(gzh)


# ==========================================================================
# charge cloud and density accumulation (density.py:58-311)
# ==========================================================================


@dataclass
class Cloud:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    w: np.ndarray
    h: np.ndarray
    dep: np.ndarray
    weight: np.ndarray
    is_macro: np.ndarray

    @property
    def volume(self):
        return self.w * self.h * self.dep

    @property
    def charge(self):
        return self.weight * self.volume

    def take(self, m):
        return Cloud(*(getattr(self, f)[m] for f in
                       ("x", "y", "z", "w", "h", "dep", "weight", "is_macro")))


def size_at_depth(w_top, h_top, w_bot, h_bot, is_macro, z, dz):
    """density.py:134-147 (Eqs. 6-7)."""
    z = np.clip(np.asarray(z, float), dz / 4, 3 * dz / 4)
    up = below_or_on_mid(z, dz)
    t = 2 * z / dz - 0.5
    wm = t * w_top + (1 - t) * w_bot
    hm = t * h_top + (1 - t) * h_bot
    return (np.where(is_macro, wm, np.where(up, w_top, w_bot)),
            np.where(is_macro, hm, np.where(up, h_top, h_bot)))


def _box(grid, cl):
    """density.py:162-169."""
    return (np.clip(cl.x - cl.w / 2, 0, grid.dx), np.clip(cl.x + cl.w / 2, 0, grid.dx),
            np.clip(cl.y - cl.h / 2, 0, grid.dy), np.clip(cl.y + cl.h / 2, 0, grid.dy),
            np.clip(cl.z - cl.dep / 2, 0, grid.dz), np.clip(cl.z + cl.dep / 2, 0, grid.dz))


def _axis_terms(lo, hi, step, n):
    """density.py:155-159 + 172-173: per offset k, (bin index, overlap length)."""
    i0 = np.clip(np.floor(lo / step).astype(np.int64), 0, n - 1)
    i1 = np.maximum(np.clip(np.ceil(hi / step).astype(np.int64) - 1, 0, n - 1), i0)
    reach = int((i1 - i0).max()) + 1 if len(i0) else 0
    out = []
    for k in range(reach):
        i = np.minimum(i0 + k, i1)
        ln = np.clip(np.minimum(hi, (i + 1) * step) - np.maximum(lo, i * step), 0, None)
        out.append((i, np.where(i0 + k <= i1, ln, 0.0)))
    return out


def overlap_terms(grid, cl):
    """density.py:176-196: every (object, bin) overlap, offset triple by triple."""
    xlo, xhi, ylo, yhi, zlo, zhi = _box(grid, cl)
    tx = _axis_terms(xlo, xhi, grid.wb, grid.nx)
    ty = _axis_terms(ylo, yhi, grid.hb, grid.ny)
    tz = _axis_terms(zlo, zhi, grid.db, grid.nz)
    for ix, wx in tx:
        for iy, wy in ty:
            wxy = wx * wy
            for iz, wz in tz:
                yield (ix * grid.ny + iy) * grid.nz + iz, wxy * wz


def direct_rho(grid, cl):
    """density.py:199-204."""
    acc = np.zeros(grid.nx * grid.ny * grid.nz)
    for flat, vol in overlap_terms(grid, cl):
        acc += np.bincount(flat, weights=cl.weight * vol, minlength=acc.size)
    return acc.reshape(grid.shape) / grid.bin_vol


def _corners(grid, cl):
    """density.py:275-288: 8 signed corners per macro, clipped to the region."""
    out = []
    for sx in (-1.0, 1.0):
        for sy in (-1.0, 1.0):
            for sz in (-1.0, 1.0):
                out.append((np.clip(cl.x + sx * cl.w / 2, 0, grid.dx),
                            np.clip(cl.y + sy * cl.h / 2, 0, grid.dy),
                            np.clip(cl.z + sz * cl.dep / 2, 0, grid.dz),
                            -sx * sy * sz))
    return out


def _stamp_iter(grid, xs, ys, zs):
    """Trilinear stamp pieces of corners (density.py:243-272, 505-530)."""
    xh, yh, zh = xs / grid.wb, ys / grid.hb, zs / grid.db
    i0, j0, k0 = (np.floor(a).astype(np.int64) for a in (xh, yh, zh))
    fx, fy, fz = xh - i0, yh - j0, zh - k0
    for bx in (0, 1):
        gi, gx = i0 + bx, (fx if bx else 1.0 - fx)
        okx = (gi >= 0) & (gi < grid.nx)
        for by in (0, 1):
            gj, gy = j0 + by, (fy if by else 1.0 - fy)
            oky = okx & (gj >= 0) & (gj < grid.ny)
            for bz in (0, 1):
                gk, gz = k0 + bz, (fz if bz else 1.0 - fz)
                ok = oky & (gk >= 0) & (gk < grid.nz)
                yield gi, gj, gk, (gx, gy, gz), ok


def macro_rho(grid, cl):
    """density.py:291-298 (Theorem 1): corner stamps + inclusive 3D prefix sum."""
    if len(cl.x) == 0:
        return np.zeros(grid.shape)
    cs = _corners(grid, cl)
    xs = np.concatenate([c[0] for c in cs])
    ys = np.concatenate([c[1] for c in cs])
    zs = np.concatenate([c[2] for c in cs])
    ws = np.concatenate([np.full(len(cl.x), c[3]) * cl.weight for c in cs])
    a = np.zeros(grid.shape)
    for gi, gj, gk, (gx, gy, gz), ok in _stamp_iter(grid, xs, ys, zs):
        if ok.any():
            np.add.at(a, (gi[ok], gj[ok], gk[ok]), (ws * gx * gy * gz)[ok])
    return np.cumsum(np.cumsum(np.cumsum(a, axis=0), axis=1), axis=2)


def rho_map(grid, cl):
    """density.py:301-311."""
    rho = np.zeros(grid.shape)
    cells = cl.take(~cl.is_macro)
    if len(cells.x):
        rho += direct_rho(grid, cells)
    mac = cl.take(cl.is_macro)
    if len(mac.x):
        rho += macro_rho(grid, mac)
    return rho


# ==========================================================================
# spectral solve (density.py:319-368)
# ==========================================================================


def potential(rho, grid):
    """density.py:319-328: DCT-II, divide by the eigenvalue, inverse."""
    coef = sfft.dctn(rho, type=2)
    return sfft.idctn(coef * grid.inv_lam, type=2), coef


def _cos_series(c, axis):
    """sum_k c_k cos(omega_k x_m) at bin centres (density.py:339-344)."""
    d = np.array(c, copy=True)
    idx = [slice(None)] * 3
    idx[axis] = slice(1, None)
    d[tuple(idx)] *= 0.5
    return sfft.dct(d, type=3, axis=axis)


def _sin_series(c, axis):
    """sum_{k>=1} c_k sin(omega_k x_m) at bin centres (density.py:347-354)."""
    n = c.shape[axis]
    d = np.zeros_like(c)
    dst_i = [slice(None)] * 3
    src_i = [slice(None)] * 3
    dst_i[axis] = slice(0, n - 1)
    src_i[axis] = slice(1, None)
    d[tuple(dst_i)] = c[tuple(src_i)] * 0.5
    return sfft.dst(d, type=3, axis=axis)


def efield(coef, grid):
    """density.py:357-368: E = -grad(phi), evaluated from true cosine-series
    coefficients a = coef / N with every index-0 plane halved."""
    a = coef / (grid.nx * grid.ny * grid.nz)
    a[0, :, :] *= 0.5
    a[:, 0, :] *= 0.5
    a[:, :, 0] *= 0.5
    base = a * grid.inv_lam
    wx, wy, wz = grid.omega
    ex = _cos_series(_cos_series(_sin_series(base * wx[:, None, None], 0), 1), 2)
    ey = _cos_series(_cos_series(_sin_series(base * wy[None, :, None], 1), 0), 2)
    ez = _cos_series(_cos_series(_sin_series(base * wz[None, None, :], 2), 0), 1)
    return ex, ey, ez


# ==========================================================================
# energy, force, overflow (density.py:376-617)
# ==========================================================================


def cell_means(grid, cl, maps):
    """density.py:376-386: overlap-weighted mean of each map over each cuboid."""
    acc = [np.zeros(len(cl.x)) for _ in maps]
    tot = np.zeros(len(cl.x))
    flat_maps = [m.reshape(-1) for m in maps]
    for flat, vol in overlap_terms(grid, cl):
        tot += vol
        for a, m in zip(acc, flat_maps):
            a += m[flat] * vol
    tot = np.maximum(tot, 1e-300)
    return [a / tot for a in acc]


def rev_cumsum3(a):
    """density.py:212-217 (adjoint of the prefix sum)."""
    for ax in range(3):
        a = np.flip(np.cumsum(np.flip(a, ax), axis=ax), ax)
    return a


def macro_means(grid, cl, smap):
    """density.py:489-530: stamp dot products against the suffix-summed map,
    divided by the unclipped cuboid volume."""
    acc = np.zeros(len(cl.x))
    for xs, ys, zs, sign in _corners(grid, cl):
        dot = np.zeros(len(xs))
        for gi, gj, gk, (gx, gy, gz), ok in _stamp_iter(grid, xs, ys, zs):
            if ok.any():
                part = np.zeros(len(xs))
                part[ok] = smap[gi[ok], gj[ok], gk[ok]] * (gx * gy * gz)[ok]
                dot += part
        acc += sign * dot
    return acc * grid.bin_vol / np.maximum(cl.volume, 1e-300)


def energy(grid, cl, phi):
    """density.py:568-579."""
    mean = np.zeros(len(cl.x))
    c = ~cl.is_macro
    if c.any():
        mean[c] = cell_means(grid, cl.take(c), (phi,))[0]
    if cl.is_macro.any():
        mean[cl.is_macro] = macro_means(grid, cl.take(cl.is_macro), rev_cumsum3(phi))
    return float((cl.charge * mean).sum())


def force(grid, cl, ex, ey, ez, freeze_z=None):
    """density.py:582-609: -2 q <E>, filler depth frozen."""
    g = np.zeros((len(cl.x), 3))
    c = ~cl.is_macro
    if c.any():
        for k, m in enumerate(cell_means(grid, cl.take(c), (ex, ey, ez))):
            g[c, k] = m
    if cl.is_macro.any():
        sub = cl.take(cl.is_macro)
        for k, m in enumerate((ex, ey, ez)):
            g[cl.is_macro, k] = macro_means(grid, sub, rev_cumsum3(m))
    g *= -2.0 * cl.charge[:, None]
    if freeze_z is not None:
        g[freeze_z, 2] = 0.0
    return g


def _axis_bins(lo, hi, step, n):
    """density.py:155-159: inclusive bin range of a clipped extent."""
    i0 = np.clip(np.floor(lo / step).astype(np.int64), 0, n - 1)
    i1 = np.maximum(np.clip(np.ceil(hi / step).astype(np.int64) - 1, 0, n - 1), i0)
    return i0, i1


def _olap(lo, hi, idx, step):
    """density.py:172-173."""
    return np.clip(np.minimum(hi, (idx + 1) * step) - np.maximum(lo, idx * step), 0, None)


def face_grad(grid, cl, phi):
    """density.py:389-441 (_direct_face_grad): d/d(center) of sum_b phi_b *
    vol(D cap b) from the two face columns of each axis; [n, 3]."""
    n = len(cl.x)
    xlo, xhi, ylo, yhi, zlo, zhi = _box(grid, cl)
    flat = phi.reshape(-1)
    out = np.zeros((n, 3))
    bounds = ((xlo, xhi, grid.wb, grid.nx), (ylo, yhi, grid.hb, grid.ny),
              (zlo, zhi, grid.db, grid.nz))
    ranges = [_axis_bins(lo, hi, st, nb) for lo, hi, st, nb in bounds]
    for axis in range(3):
        lo, hi, step, nb = bounds[axis]
        f_hi = np.clip(np.floor(hi / step).astype(np.int64), 0, nb - 1)  # density.py:392-394
        f_lo = np.clip(np.floor(lo / step).astype(np.int64), 0, nb - 1)
        o1, o2 = [a for a in (0, 1, 2) if a != axis]
        (l1, h1, s1, _), (l2, h2, s2, _) = bounds[o1], bounds[o2]
        (i10, i11), (i20, i21) = ranges[o1], ranges[o2]
        acc = np.zeros(n)
        for d1 in range(int((i11 - i10).max(initial=-1)) + 1):
            b1 = np.minimum(i10 + d1, i11)
            w1 = np.where(i10 + d1 <= i11, _olap(l1, h1, b1, s1), 0.0)
            for d2 in range(int((i21 - i20).max(initial=-1)) + 1):
                b2 = np.minimum(i20 + d2, i21)
                w2 = np.where(i20 + d2 <= i21, _olap(l2, h2, b2, s2), 0.0)
                w12 = w1 * w2
                idx = [None, None, None]
                idx[o1], idx[o2] = b1, b2
                idx[axis] = f_hi
                fhi = (idx[0] * grid.ny + idx[1]) * grid.nz + idx[2]
                idx[axis] = f_lo
                flo = (idx[0] * grid.ny + idx[1]) * grid.nz + idx[2]
                acc += (flat[fhi] - flat[flo]) * w12
        out[:, axis] = acc
    return out


def stamp_face_grad(grid, cl, sphi):
    """density.py:444-486 (_stamp_face_grad): macro gradient from corner stamps
    differentiated along the gradient axis, against the suffix-summed phi."""
    n = len(cl.x)
    out = np.zeros((n, 3))
    steps = (grid.wb, grid.hb, grid.db)
    nbins = (grid.nx, grid.ny, grid.nz)
    extents = (grid.dx, grid.dy, grid.dz)
    half = (cl.w / 2, cl.h / 2, cl.dep / 2)
    centers = (cl.x, cl.y, cl.z)
    for axis in range(3):
        acc = np.zeros(n)
        for sx in (-1.0, 1.0):
            for sy in (-1.0, 1.0):
                for sz in (-1.0, 1.0):
                    sign = -sx * sy * sz
                    sigma = (sx, sy, sz)
                    coords = [np.clip(centers[a] + sigma[a] * half[a], 0, extents[a])
                              for a in range(3)]
                    stamps = []
                    for a in range(3):
                        base = coords[a] / steps[a]
                        i0 = np.floor(base).astype(np.int64)
                        frac = base - i0
                        if a == axis:
                            stamps.append([(i0, -1.0 / steps[a]), (i0 + 1, 1.0 / steps[a])])
                        else:
                            stamps.append([(i0, 1.0 - frac), (i0 + 1, frac)])
                    for g0, v0 in stamps[0]:
                        ok0 = (g0 >= 0) & (g0 < nbins[0])
                        for g1, v1 in stamps[1]:
                            ok1 = ok0 & (g1 >= 0) & (g1 < nbins[1])
                            for g2, v2 in stamps[2]:
                                ok = ok1 & (g2 >= 0) & (g2 < nbins[2])
                                if not ok.any():
                                    continue
                                val = np.zeros(n)
                                val[ok] = sphi[g0[ok], g1[ok], g2[ok]]
                                acc += sign * val * (v0 * v1 * np.asarray(v2))
        out[:, axis] = acc * grid.bin_vol
    return out


def energy_and_gradient(grid, cl, phi, freeze_z=None):
    """density.py:533-565 (density_energy_and_gradient): U = sum q phibar and its
    exact gradient 2 w sum_b phi_b dvol/dc (cells: face form; macros: stamps)."""
    n = len(cl.x)
    grad = np.zeros((n, 3))
    phibar = np.zeros(n)
    c = ~cl.is_macro
    if c.any():
        sub = cl.take(c)
        phibar[c] = cell_means(grid, sub, (phi,))[0]
        grad[c] = face_grad(grid, sub, phi) * (2.0 * sub.weight[:, None])
    if cl.is_macro.any():
        sub = cl.take(cl.is_macro)
        sphi = rev_cumsum3(phi)
        phibar[cl.is_macro] = macro_means(grid, sub, sphi)
        grad[cl.is_macro] = stamp_face_grad(grid, sub, sphi) * (2.0 * sub.weight[:, None])
    energy = float((cl.charge * phibar).sum())
    if freeze_z is not None:
        grad[freeze_z, 2] = 0.0
    return energy, grad


def overflow_of(rho, grid, rho_t, mv):
    """density.py:612-617."""
    if mv <= 0:
        return 0.0
    return float(np.clip(rho - rho_t, 0, None).sum() * grid.bin_vol / mv)


# ==========================================================================
# GP setup, preconditioner, optimizer, loop (gp.py:75-455)
# ==========================================================================


@dataclass
class Fill:
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


def fillers_for(design, grid, rng):
    """gp.py:129-139 + density.py:107-131 (rng draws in the reference order)."""
    arr = design.arrays()
    cells = ~arr.is_macro
    hint = float(np.median(arr.w_bot[cells] * arr.h_bot[cells])) if cells.any() \
        else (design.die.width / 32) ** 2
    dx, dy, dz = design.die.width, design.die.height, grid.dz
    parts = []
    for die, u in ((0, design.die.max_util_bottom), (1, design.die.max_util_top)):
        area = dx * dy * (1.0 - u)
        if area <= 0:
            continue
        s_hint = max(np.sqrt(hint), 1e-9)
        cnt = int(np.clip(round(area / s_hint ** 2), 1, 20000))
        side = np.sqrt(area / cnt)
        xs = rng.uniform(side / 2, dx - side / 2, cnt)
        ys = rng.uniform(side / 2, dy - side / 2, cnt)
        parts.append((xs, ys, np.full(cnt, dz / 4 if die == 0 else 3 * dz / 4),
                      np.full(cnt, die, np.int8), np.full(cnt, side), np.full(cnt, side)))
    if not parts:
        e = np.zeros(0)
        return Fill(e, e, e, np.zeros(0, np.int8), e, e, dz / 2)
    cat = [np.concatenate([p[i] for p in parts]) for i in range(6)]
    return Fill(*cat, dz / 2)


def grid_for(design, cfg):
    """gp.py:75-87."""
    n = max(design.n_insts, 1)
    if cfg.grid_nx is not None:
        nx, ny = cfg.grid_nx, (cfg.grid_ny or cfg.grid_nx)
    else:
        k = 3
        while (2 ** (k + 1)) ** 2 <= n / 4 and 2 ** (k + 1) <= 128:
            k += 1
        nx = ny = 2 ** k
    return Grid(design.die.width, design.die.height, nx, ny, cfg.nz)


def start_state(design, grid, cfg, rng):
    """gp.py:115-126: (x, y, z, rot) around the centre with seeded jitter."""
    n = design.n_insts
    die = design.die
    x = np.full(n, die.width / 2) + rng.normal(0, cfg.jitter_frac * die.width, n)
    y = np.full(n, die.height / 2) + rng.normal(0, cfg.jitter_frac * die.height, n)
    z = np.full(n, grid.dz / 2) + rng.normal(0, cfg.jitter_frac * grid.dz, n)
    arr = design.arrays()
    x = np.clip(x, arr.w_bot / 2, die.width - arr.w_bot / 2)
    y = np.clip(y, arr.h_bot / 2, die.height - arr.h_bot / 2)
    z = np.clip(z, grid.dz / 4, 3 * grid.dz / 4)
    return x, y, z, np.zeros(n, dtype=np.int64)


def alpha_of(design, dz, cfg):
    """gp.py:90-107."""
    if cfg.alpha is not None:
        return cfg.alpha
    die, hbt = design.die, design.hbt
    eta = 2 * hbt.pitch / (die.row_height_top + die.row_height_bottom)
    arg = max(90 * hbt.cost * eta - 1, 1 + 1e-6)
    lg = math.log(arg) if cfg.log_base is None else math.log(arg, cfg.log_base)
    return max(cfg.alpha0 * (die.width * eta ** 2 / dz) * lg,
               cfg.cut_cost_factor * hbt.cost / (dz / 2))


def precond(g, lam, q, deg, macro):
    """gp.py:142-147 (Eq. 19)."""
    div = lam * np.asarray(q, float)
    div = div + np.where(macro, np.asarray(deg, float), 0.0)
    div = np.maximum(div, 1.0)
    return g / div[..., None], div


def lam0(wl_norm, dens_norm, scale=1e-3):
    """gp.py:150-153."""
    return scale if (wl_norm <= 0 or dens_norm <= 0) else scale * wl_norm / dens_norm


def mu_of(prev, cur, cfg):
    """gp.py:156-168."""
    drop = prev - cur
    if drop < 0:
        mu = cfg.mu_min
    elif drop >= 2e-3:
        mu = cfg.mu_min + 0.01
    elif drop >= 5e-4:
        mu = (cfg.mu_min + cfg.mu_max) / 2
    else:
        mu = cfg.mu_max
    return min(max(mu, cfg.mu_min), cfg.mu_max)


def gamma_at(db, it, max_iters, cfg):
    """gp.py:171-175."""
    t = min(1.0, it / max(max_iters - 1, 1))
    g0 = cfg.gamma_start_factor * db
    g1 = cfg.gamma_end_factor * db
    return g0 * (g1 / g0) ** t


def clamp_span(v, size, extent):
    """gp.py:344-348."""
    lo = size / 2
    hi = extent - size / 2
    mid = np.minimum(lo, hi) + np.abs(hi - lo) / 2
    return np.where(lo <= hi, np.clip(v, np.minimum(lo, hi), np.maximum(lo, hi)), mid)


class StepUnderflow(RuntimeError):
    pass


class Nesterov:
    """gp.py:178-227: Nesterov with a clipped Barzilai-Borwein step."""

    def __init__(self, x0, project=None, min_step=1e-18):
        self.project = project or (lambda p: p)
        self.u = self.project(np.array(x0, dtype=float))
        self.v = self.u.copy()
        self.a = 1.0
        self.step = None
        self.min_step = min_step
        self.prev_v = None
        self.prev_g = None

    def advance(self, g, step_scale=1.0, g_prev_reval=None):
        ref = g_prev_reval if g_prev_reval is not None else self.prev_g
        if self.step is None or self.prev_v is None or ref is None:
            if self.step is None:
                gm = float(np.abs(g).max(initial=0.0))
                self.step = 1.0 if gm == 0 else step_scale / gm
        else:
            den = float(np.linalg.norm(g - ref))
            if den > 0:
                bb = float(np.linalg.norm(self.v - self.prev_v)) / den
                self.step = float(np.clip(bb, self.step / 4, self.step * 4))
        if not np.isfinite(self.step) or self.step <= self.min_step:
            raise StepUnderflow(f"step size underflow ({self.step!r})")
        self.prev_v = self.v.copy()
        self.prev_g = np.array(g, dtype=float, copy=True)
        u1 = self.project(self.v - self.step * g)
        a1 = (1 + math.sqrt(4 * self.a ** 2 + 1)) / 2
        self.v = self.project(u1 + (self.a - 1) / a1 * (u1 - self.u))
        self.u = u1
        self.a = a1
        return self.u


@dataclass
class Eval:
    wl_grad: np.ndarray
    dens_grad: np.ndarray
    total: np.ndarray
    divisors: np.ndarray
    value: float
    wl_value: float
    energy: float
    parts: dict = dc_field(default_factory=dict)


class Problem:
    """gp.py:235-341: one 3D GP evaluation context (instances then fillers)."""

    def __init__(self, design, grid, fill, cfg, rot):
        self.design, self.grid, self.fill, self.cfg = design, grid, fill, cfg
        self.rot = np.asarray(rot)
        a = self.arr = design.arrays()
        self.n_inst = design.n_insts
        self.n_fill = fill.count
        self.n_obj = self.n_inst + self.n_fill
        self.alpha = alpha_of(design, grid.dz, cfg)
        odd = (self.rot % 4) % 2 == 1
        self.w_top, self.h_top = np.where(odd, a.h_top, a.w_top), np.where(odd, a.w_top, a.h_top)
        self.w_bot, self.h_bot = np.where(odd, a.h_bot, a.w_bot), np.where(odd, a.w_bot, a.h_bot)
        self.is_macro_obj = np.r_[a.is_macro, np.zeros(self.n_fill, bool)]
        self.degree_obj = np.r_[a.pin_degree, np.zeros(self.n_fill)]
        self.freeze_z = np.r_[np.zeros(self.n_inst, bool), np.ones(self.n_fill, bool)]
        self.weight = np.r_[np.where(a.is_macro, cfg.target_density, 1.0), np.ones(self.n_fill)]
        w, h = size_at_depth(self.w_top, self.h_top, self.w_bot, self.h_bot, a.is_macro,
                             np.full(self.n_inst, grid.dz / 2), grid.dz)
        self.movable_volume = float((w * h).sum() * grid.dz / 2)

    def cloud(self, pos):
        w, h = size_at_depth(self.w_top, self.h_top, self.w_bot, self.h_bot,
                             self.arr.is_macro, pos[: self.n_inst, 2], self.grid.dz)
        return Cloud(pos[:, 0], pos[:, 1], pos[:, 2], np.r_[w, self.fill.w],
                     np.r_[h, self.fill.h], np.full(self.n_obj, self.grid.dz / 2),
                     self.weight, self.is_macro_obj)

    def project(self, pos):
        g, dz, n = self.grid, self.grid.dz, self.n_inst
        out = pos.copy()
        z = np.clip(out[:n, 2], dz / 4, 3 * dz / 4)
        out[:n, 2] = z
        w, h = size_at_depth(self.w_top, self.h_top, self.w_bot, self.h_bot,
                             self.arr.is_macro, z, dz)
        out[:n, 0] = clamp_span(out[:n, 0], w, g.dx)
        out[:n, 1] = clamp_span(out[:n, 1], h, g.dy)
        out[n:, 0] = clamp_span(out[n:, 0], self.fill.w, g.dx)
        out[n:, 1] = clamp_span(out[n:, 1], self.fill.h, g.dy)
        out[n:, 2] = self.fill.z
        return out

    def evaluate(self, pos, lam, gamma, keep=False):
        g, a, n = self.grid, self.arr, self.n_inst
        x, y, z = pos[:n, 0], pos[:n, 1], pos[:n, 2]
        px, py, pz, top = pins_at(a, x, y, z, self.rot, g.dz)
        bx = Boxes(a.pin_net, a.n_net, px, top)
        by = Boxes(a.pin_net, a.n_net, py, top)
        wl_bi, gxp, gyp = planar_wl(a.pin_net, a.n_net, px, py, top, gamma, bx, by)
        cut, gcp = zcut(a.pin_net, a.n_net, pz, gamma)
        gx = np.bincount(a.pin_inst, weights=gxp, minlength=n)
        gy = np.bincount(a.pin_inst, weights=gyp, minlength=n)
        gzh = np.bincount(a.pin_inst, weights=gcp, minlength=n)
        gzb = fd_depth_grad(a.net_ptr, a.pin_net, a.pin_inst, n, px, py, top, g.dz,
                            a.net_has_dup_inst, bx, by)
        gz = normalize_depth(gx, gy, gzb, gzh, self.alpha)
        wl_grad = np.zeros((self.n_obj, 3))
        wl_grad[:n, 0], wl_grad[:n, 1], wl_grad[:n, 2] = gx, gy, gz
        cl = self.cloud(pos)
        rho = rho_map(g, cl)
        phi, coef = potential(rho, g)
        ex, ey, ez = efield(coef, g)
        en = energy(g, cl, phi)
        dg = force(g, cl, ex, ey, ez, freeze_z=self.freeze_z)
        value = wl_bi + self.alpha * cut + lam * en
        total = wl_grad + lam * dg
        if not np.isfinite(value) or not np.all(np.isfinite(total)):
            raise FloatingPointError("non-finite objective or gradient")
        _, div = precond(total, lam, cl.charge, self.degree_obj, self.is_macro_obj)
        ev = Eval(wl_grad, dg, total, div, value, wl_bi + self.alpha * cut, en)
        if keep:
            ev.parts = dict(px=px, py=py, pz=pz, top=top, bx=bx, by=by, wl_bi=wl_bi,
                            cut=cut, gx=gx, gy=gy, gzh=gzh, gzb=gzb, rho=rho, phi=phi,
                            coef=coef, ex=ex, ey=ey, ez=ez, cloud=cl)
        ovfl = overflow_of(rho, g, self.cfg.target_density, self.movable_volume)
        exact = float(bx.bistratal().sum() + by.bistratal().sum())
        dt = below_or_on_mid(z, g.dz)[a.pin_inst].astype(np.int8)
        hi = np.zeros(a.n_net, np.int8)
        lo = np.ones(a.n_net, np.int8)
        np.maximum.at(hi, a.pin_net, dt)
        np.minimum.at(lo, a.pin_net, dt)
        return ev, ovfl, exact, int((hi > lo).sum())


@dataclass
class LoopInfo:
    iterations: int = 0
    final_overflow: float = math.inf
    diverged: bool = False
    wirelength: float = 0.0
    hbt_count: int = 0


def run_loop(design, x, y, z, rot, fill, cfg, grid, log=None, iter_limit=None):
    """gp.py:359-455 (run_gp3d) on already-built fillers.  ``iter_limit`` stops
    early without changing the schedule (used to bound CPU-baseline samples).
    Returns (inst pos [I,3] after the epilogue, filler xy, info)."""
    prob = Problem(design, grid, fill, cfg, rot)
    n = prob.n_inst
    pos0 = np.zeros((prob.n_obj, 3))
    pos0[:n] = np.c_[x, y, z]
    pos0[n:] = np.c_[fill.x, fill.y, fill.z]
    opt = Nesterov(pos0, project=prob.project)
    info = LoopInfo()
    lam = None
    best = (math.inf, math.inf)
    best_pos = opt.u.copy()
    prev_ovfl = math.inf
    rise = 0
    prev_value = math.inf
    last_mu = 1.0
    hist = []
    prev_raw = None
    limit = cfg.max_iters if iter_limit is None else min(iter_limit, cfg.max_iters)
    for it in range(limit):
        gamma = gamma_at(grid.db, it, cfg.max_iters, cfg)
        try:
            ev, ovfl, exact, ncross = prob.evaluate(opt.v, lam or 0.0, gamma)
        except FloatingPointError:
            info.diverged = True
            break
        if lam is None:
            lam = lam0(np.abs(ev.wl_grad).sum(), np.abs(ev.dens_grad).sum())
            ev.value = ev.wl_value + lam * ev.energy
            ev.total = ev.wl_grad + lam * ev.dens_grad
        if log is not None:
            log.append((it, exact, ncross, ovfl))
        info.iterations = it + 1
        info.final_overflow = ovfl
        info.wirelength = exact
        info.hbt_count = ncross
        key = (max(ovfl - cfg.stop_overflow, 0.0), ev.value)
        if key < best:
            best = key
            best_pos = opt.u.copy()
        if ovfl <= cfg.stop_overflow:
            break
        rise = rise + 1 if ev.value > prev_value * last_mu else 0
        prev_value = ev.value
        hist.append(ovfl)
        if rise >= cfg.divergence_window:
            win = hist[-cfg.divergence_window:]
            if win[0] - win[-1] < 1e-3:
                info.diverged = True
                break
        q = prob.cloud(opt.v).charge
        pre, _ = precond(ev.total, lam, q, prob.degree_obj, prob.is_macro_obj)
        pre_prev = None
        if prev_raw is not None:
            pre_prev, _ = precond(prev_raw[0] + lam * prev_raw[1], lam, prev_raw[2],
                                  prob.degree_obj, prob.is_macro_obj)
        prev_raw = (ev.wl_grad, ev.dens_grad, q)
        try:
            opt.advance(pre, step_scale=grid.wb, g_prev_reval=pre_prev)
        except StepUnderflow:
            info.diverged = True
            break
        last_mu = mu_of(prev_ovfl, ovfl, cfg)
        lam *= last_mu
        prev_ovfl = ovfl
    final = opt.u if info.final_overflow <= cfg.stop_overflow else best_pos
    final = prob.project(final)
    zz = final[:n, 2]
    zz = np.where(below_or_on_mid(zz, grid.dz), 3 * grid.dz / 4, grid.dz / 4)
    inst = np.c_[final[:n, 0], final[:n, 1], zz]
    return inst, final[n:, :2].copy(), info


@dataclass
class Cfg:
    """Field-for-field mirror of ``GpConfig`` (gp.py:30-50)."""

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


# ==========================================================================
# multi-die 2D GP (gp.py:463-690)
# ==========================================================================


def optimal_region(top_box, bot_box):
    """wirelength.py:153-164."""
    out = []
    for a in (0, 2):
        lo = max(top_box[a], bot_box[a])
        hi = min(top_box[a + 1], bot_box[a + 1])
        out.extend((min(lo, hi), max(lo, hi)))
    return tuple(out)


def hbt_centers(arr, x, y, z, rot, dz):
    """wirelength.py:325-342 (optimal_hbt_centers): {net: (cx, cy)} per
    crossing net, the centre of the zero-added-wirelength region."""
    px, py, _, top = pins_at(arr, x, y, z, rot, dz)
    bx = Boxes(arr.pin_net, arr.n_net, px, top)
    by = Boxes(arr.pin_net, arr.n_net, py, top)
    crossing = np.flatnonzero((bx.cnt[:, 0] > 0) & (bx.cnt[:, 1] > 0))
    out = {}
    for j in crossing:
        r = optimal_region((bx.min1[j, 1], bx.max1[j, 1], by.min1[j, 1], by.max1[j, 1]),
                           (bx.min1[j, 0], bx.max1[j, 0], by.min1[j, 0], by.max1[j, 0]))
        out[int(j)] = ((r[0] + r[1]) / 2, (r[2] + r[3]) / 2)
    return out


class Gp2d:
    """gp.py:463-528 (Gp2dProblem): three nz = 1 grids (bottom, top, terminal
    layer), the augmented pin list in which each HBT joins both partial nets of
    its crossing net, and pin offsets frozen at the partition."""

    def __init__(self, design, cfg, delta, rot, n_grid):
        arr = design.arrays()
        self.arr = arr
        self.delta = np.asarray(delta)
        die = design.die
        self.grids = [Grid(die.width, die.height, n_grid, n_grid, 1) for _ in range(3)]
        pd = self.delta[arr.pin_inst]
        mx = np.zeros(design.n_nets, dtype=np.int8)
        mn = np.ones(design.n_nets, dtype=np.int8)
        np.maximum.at(mx, arr.pin_net, pd)
        np.minimum.at(mn, arr.pin_net, pd)
        self.crossing = np.flatnonzero(mx > mn)
        self.n_inst = design.n_insts
        self.n_hbt = len(self.crossing)
        self.n_core = self.n_inst + self.n_hbt
        pin_net = np.r_[arr.pin_net, self.crossing, self.crossing]
        pin_obj = np.r_[arr.pin_inst, self.n_inst + np.arange(self.n_hbt),
                        self.n_inst + np.arange(self.n_hbt)]
        top = np.r_[pd == 1, np.ones(self.n_hbt, bool), np.zeros(self.n_hbt, bool)]
        order = np.argsort(pin_net, kind="stable")
        self.pin_net, self.pin_obj, self.pin_top = pin_net[order], pin_obj[order], top[order]
        cnt = np.bincount(self.pin_net, minlength=design.n_nets)
        self.net_ptr = np.zeros(design.n_nets + 1, dtype=np.int64)
        np.cumsum(cnt, out=self.net_ptr[1:])
        wt, ht = turn_offsets_dims(arr.w_top, arr.h_top, rot)
        wb, hb = turn_offsets_dims(arr.w_bot, arr.h_bot, rot)
        self.inst_w = np.where(self.delta == 1, wt, wb)
        self.inst_h = np.where(self.delta == 1, ht, hb)
        self.hbt_size = design.hbt.pitch + design.hbt.spacing
        q = np.asarray(rot)[arr.pin_inst]
        rx_t, ry_t = turn_offsets(arr.ox_top, arr.oy_top, q)
        rx_b, ry_b = turn_offsets(arr.ox_bot, arr.oy_bot, q)
        it = pd == 1
        self.pin_ox = np.r_[np.where(it, rx_t, rx_b), np.zeros(2 * self.n_hbt)][order]
        self.pin_oy = np.r_[np.where(it, ry_t, ry_b), np.zeros(2 * self.n_hbt)][order]


def turn_offsets_dims(w, h, q):
    """model.py:292-295 (rotated_dims): w/h swap on odd quarter turns."""
    odd = (np.asarray(q) % 4) % 2 == 1
    return np.where(odd, h, w), np.where(odd, w, h)


def gp2d_grid_n(n_insts):
    """gp.py:536-539."""
    n = max(n_insts, 1)
    k = 2
    while (2 ** (k + 1)) ** 2 <= n / 4 and 2 ** (k + 1) <= 128:
        k += 1
    return 2 ** k


def gp2d_run(design, x, y, z, rot, dz, cfg, rng, log=None):
    """gp.py:531-690 (run_gp2d_multi): returns (x, y, info, hbt_centers)."""
    delta = (np.asarray(z) - dz / 2 > 0).astype(np.int8)
    prob = Gp2d(design, cfg, delta, rot, gp2d_grid_n(design.n_insts))
    die = design.die
    grids = prob.grids
    arr = prob.arr
    cells = ~arr.is_macro
    hint = float(np.median(arr.w_bot[cells] * arr.h_bot[cells])) if cells.any() \
        else (die.width / 32) ** 2
    fxy, fwh, flay = [], [], []
    for layer, u in ((0, die.max_util_bottom), (1, die.max_util_top)):  # gp.py:552-562
        area = die.width * die.height * (1 - u)
        if area <= 0:
            continue
        count = int(np.clip(round(area / max(hint, 1e-9)), 1, 20000))
        side = math.sqrt(area / count)
        fxy.append(np.c_[rng.uniform(side / 2, die.width - side / 2, count),
                         rng.uniform(side / 2, die.height - side / 2, count)])
        fwh.append(np.full((count, 2), side))
        flay.append(np.full(count, layer))
    fx = np.concatenate(fxy) if fxy else np.zeros((0, 2))
    fwh = np.concatenate(fwh) if fwh else np.zeros((0, 2))
    flay = np.concatenate(flay) if flay else np.zeros(0, int)
    n_core = prob.n_core
    n_obj = n_core + len(fx)
    pos = np.zeros((n_obj, 2))
    pos[: prob.n_inst] = np.c_[x, y]
    cen = hbt_centers(arr, x, y, z, rot, dz)
    for t, j in enumerate(prob.crossing):
        pos[prob.n_inst + t] = cen.get(int(j), (die.width / 2, die.height / 2))
    pos[n_core:] = fx
    size_w = np.r_[prob.inst_w, np.full(prob.n_hbt, prob.hbt_size), fwh[:, 0]]
    size_h = np.r_[prob.inst_h, np.full(prob.n_hbt, prob.hbt_size), fwh[:, 1]]
    obj_layer = np.r_[delta.astype(int), np.full(prob.n_hbt, 2), flay]
    is_macro = np.r_[arr.is_macro, np.zeros(prob.n_hbt + len(fx), bool)]
    degree = np.r_[arr.pin_degree, np.full(prob.n_hbt, 2.0), np.zeros(len(fx))]
    is_filler = np.r_[np.zeros(n_core, bool), np.ones(len(fx), bool)]

    def project(p):
        out = p.copy()
        out[:, 0] = clamp_span(out[:, 0], size_w, die.width)
        out[:, 1] = clamp_span(out[:, 1], size_h, die.height)
        return out

    mv = [float((size_w[m] * size_h[m]).sum() * grids[l].db)
          for l, m in enumerate([(obj_layer == l) & ~is_filler for l in range(3)])]
    seg = prob.pin_net * 2 + prob.pin_top.astype(np.int64)
    n_net = len(prob.net_ptr) - 1

    def evaluate(p, gamma):  # gp.py:586-626
        px = p[prob.pin_obj, 0] + prob.pin_ox
        py = p[prob.pin_obj, 1] + prob.pin_oy
        val = 0.0
        gxp = np.zeros(len(px))
        gyp = np.zeros(len(px))
        for c, gp_ in ((px, gxp), (py, gyp)):
            v, g = wa_segments(seg, 2 * n_net, c, gamma)
            val += float(v.sum())
            gp_ += g
        wl_g = np.c_[np.bincount(prob.pin_obj, weights=gxp, minlength=n_obj),
                     np.bincount(prob.pin_obj, weights=gyp, minlength=n_obj)]
        dg = np.zeros((n_obj, 2))
        ovfls = []
        for layer in range(3):
            m = obj_layer == layer
            g = grids[layer]
            if not m.any():
                ovfls.append(0.0)
                continue
            k = int(m.sum())
            cl = Cloud(p[m, 0], p[m, 1], np.full(k, g.dz / 2), size_w[m], size_h[m],
                       np.full(k, g.dz), np.where(is_macro[m], cfg.target_density, 1.0),
                       is_macro[m])
            rho = rho_map(g, cl)
            phi, coef = potential(rho, g)
            ex, ey, _ = efield(coef, g)
            dg[m] = force(g, cl, ex, ey, np.zeros_like(phi))[:, :2]
            ovfls.append(overflow_of(rho, g, cfg.target_density, mv[layer]))
        return val, wl_g, dg, ovfls

    opt = Nesterov(pos, project=project)
    info = LoopInfo()
    lams = None
    charges = size_w * size_h * grids[0].db
    prev = [math.inf] * 3
    prev_raw = None
    for it in range(cfg.max_iters):  # gp.py:637-681
        gamma = gamma_at(grids[0].db, it, cfg.max_iters, cfg)
        val, wl_g, dg, ovfls = evaluate(opt.v, gamma)
        if lams is None:
            lams = [lam0(np.abs(wl_g[obj_layer == l]).sum(), np.abs(dg[obj_layer == l]).sum())
                    for l in range(3)]
        worst = max(ovfls)
        info.iterations = it + 1
        info.final_overflow = worst
        if log is not None:
            log.append((it, val, prob.n_hbt, worst))
        if worst <= cfg.stop_overflow:
            break
        lam_obj = np.array([lams[l] for l in obj_layer])
        total = wl_g + lam_obj[:, None] * dg
        pre, _ = precond(total, 1.0, lam_obj * charges, degree, is_macro)
        pre_prev = None
        if prev_raw is not None:
            pre_prev, _ = precond(prev_raw[0] + lam_obj[:, None] * prev_raw[1], 1.0,
                                  lam_obj * charges, degree, is_macro)
        prev_raw = (wl_g, dg)
        try:
            opt.advance(pre, step_scale=grids[0].wb, g_prev_reval=pre_prev)
        except StepUnderflow:
            info.diverged = True
            break
        for l in range(3):
            lams[l] *= mu_of(prev[l], ovfls[l], cfg)
            prev[l] = ovfls[l]
    final = project(opt.u)
    centers = {int(j): (float(final[prob.n_inst + t, 0]), float(final[prob.n_inst + t, 1]))
               for t, j in enumerate(prob.crossing)}
    return final[: prob.n_inst, 0].copy(), final[: prob.n_inst, 1].copy(), info, centers


# ==========================================================================
# solution score (model.py:364-400)
# ==========================================================================


def score(arr, hbt_pitch, hbt_cost, die, x, y, rot, hbt_xy):
    """evaluate_score(design, sol, allow_illegal=True) on flat arrays: die-to-die
    HPWL (per die, pins at lower-left + rotated half size + rotated offset,
    the HBT centre joining both partial nets of its net) + cost * #HBTs.
    Returns (hpwl, hbt_count, raw_score)."""
    half = hbt_pitch / 2
    q = np.asarray(rot)[arr.pin_inst]
    d = np.asarray(die)[arr.pin_inst]
    rxt, ryt = turn_offsets(arr.ox_top, arr.oy_top, q)
    rxb, ryb = turn_offsets(arr.ox_bot, arr.oy_bot, q)
    wt, ht = turn_offsets_dims(arr.w_top, arr.h_top, rot)
    wb, hb = turn_offsets_dims(arr.w_bot, arr.h_bot, rot)
    top = np.asarray(die) == 1
    w = np.where(top, wt, wb)[arr.pin_inst]
    h = np.where(top, ht, hb)[arr.pin_inst]
    px = np.asarray(x)[arr.pin_inst] + w / 2 + np.where(d == 1, rxt, rxb)  # model.py:352-361
    py = np.asarray(y)[arr.pin_inst] + h / 2 + np.where(d == 1, ryt, ryb)
    hpwl, count = 0.0, 0
    for j in range(arr.n_net):
        b, e = arr.net_ptr[j], arr.net_ptr[j + 1]
        xs = {0: list(px[b:e][d[b:e] == 0]), 1: list(px[b:e][d[b:e] == 1])}
        ys = {0: list(py[b:e][d[b:e] == 0]), 1: list(py[b:e][d[b:e] == 1])}
        crossing = bool(xs[0]) and bool(xs[1])
        t = hbt_xy.get(j)
        if t is not None:
            count += 1
            cx, cy = t[0] + half, t[1] + half
            for k in (0, 1):
                if crossing or xs[k]:
                    xs[k].append(cx)
                    ys[k].append(cy)
        for k in (0, 1):
            if xs[k]:
                hpwl += max(xs[k]) - min(xs[k]) + max(ys[k]) - min(ys[k])
    return hpwl, count, hpwl + hbt_cost * count
