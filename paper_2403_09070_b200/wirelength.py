"""Drop-in of ``place3d.wirelength`` on the B200 (K1 kernels of libp3d.so).

Same function names, argument meaning and return shapes as
``pkg/src/place3d/wirelength.py``; arrays come back as CUDA ``torch.Tensor``s
(float64) instead of numpy arrays, scalars as Python floats.  Inputs may be
numpy arrays or tensors.  The reference semantics each function keeps are
cited per function.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .model import NetlistArrays, net_dup_flags, partition_from_z, rotate_offsets

_SCR = 8 + 6 * 2048


@dataclass
class NetTopology:
    """CSR pin layout (wirelength.py:30-47).  ``device()`` stages the derived
    layouts the kernels use: degree-grouped net order, owner-sorted pin slots."""

    net_ptr: object
    pin_net: object
    pin_inst: object
    n_obj: int

    @property
    def n_net(self):
        return len(self.net_ptr) - 1

    @property
    def n_pin(self):
        return len(self.pin_net)

    @classmethod
    def from_arrays(cls, arrays: NetlistArrays):
        return cls(arrays.net_ptr, arrays.pin_net, arrays.pin_inst, arrays.n_inst)

    def device(self, net_has_dup=None):
        key = None if net_has_dup is None else id(net_has_dup)
        cache = getattr(self, "_dev_cache", None)
        if cache is not None and cache[0] == key:
            return cache[1]
        d = DeviceTopology(np.asarray(self.net_ptr), np.asarray(self.pin_inst), int(self.n_obj),
                           net_has_dup)
        self._dev_cache = (key, d)
        return d


class DeviceTopology:
    """Device-resident topology + the ctypes ``p3d_topology`` pointing at it."""

    def __init__(self, net_ptr, pin_inst, n_obj, net_has_dup=None):
        net_ptr = np.asarray(net_ptr, dtype=np.int64)
        pin_inst = np.asarray(pin_inst, dtype=np.int64)
        n_net = len(net_ptr) - 1
        n_pin = len(pin_inst)
        if n_pin >= 2 ** 31 - 1 or n_obj >= 2 ** 31 - 1:
            raise ValueError("more than 2^31 pins/objects is not supported")
        if net_has_dup is None:
            net_has_dup = net_dup_flags(net_ptr, pin_inst)
        deg = np.diff(net_ptr)
        order = _dev.stable_argsort(deg)
        slot_order = _dev.stable_argsort(pin_inst)
        slot = np.empty(n_pin, dtype=np.int64)
        slot[slot_order] = np.arange(n_pin)
        optr = np.zeros(n_obj + 1, dtype=np.int64)
        if n_pin:
            np.cumsum(np.bincount(pin_inst, minlength=n_obj), out=optr[1:])
        keep = self.keep = _dev.Keep()
        self.net_ptr = _dev.i32(net_ptr)
        self.pin_inst = _dev.i32(pin_inst)
        self.net_dup = _dev.u8(np.asarray(net_has_dup, dtype=bool))
        self.net_order = _dev.i32(order)
        self.pin_slot = _dev.i32(slot)
        self.obj_slot_ptr = _dev.i32(optr)
        self.n_net, self.n_pin, self.n_obj = n_net, n_pin, n_obj
        t = _lib.Topology()
        t.n_net, t.n_pin, t.n_obj = n_net, n_pin, n_obj
        t.net_ptr = keep(self.net_ptr)
        t.pin_inst = keep(self.pin_inst) if n_pin else None
        t.net_dup = keep(self.net_dup) if n_net else None
        t.net_order = keep(self.net_order) if n_net else None
        t.pin_slot = keep(self.pin_slot) if n_pin else None
        t.obj_slot_ptr = keep(self.obj_slot_ptr)
        self.struct = t


def _topo(topo):
    return topo.device() if isinstance(topo, NetTopology) else topo


def _flags(on_top):
    return _dev.u8(on_top.to(torch.bool) if isinstance(on_top, torch.Tensor) else np.asarray(on_top, bool))


# ---------------------------------------------------------------------------


def partial_hpwl(values):
    """max - min of a coordinate set; empty spans 0 (wirelength.py:50-55)."""
    v = _dev.f64(np.asarray(values, dtype=float) if not isinstance(values, torch.Tensor) else values)
    if v.numel() == 0:
        return 0.0
    return float((v.max() - v.min()).item())


def wa_smooth(values, gamma):
    """WA smoothed span and gradient of one coordinate set (wirelength.py:58-73),
    evaluated by the K1 kernel as a single-net z-span."""
    host = not isinstance(values, torch.Tensor)
    v = _dev.f64(np.asarray(values, dtype=float) if host else values)
    n = v.numel()
    if n == 0:
        return 0.0, (np.zeros(0) if host else torch.zeros(0, dtype=torch.float64, device="cuda"))
    topo = NetTopology(np.array([0, n]), np.zeros(n, np.int64), np.arange(n), n)
    val, grad = z_cut_penalty(topo, v, gamma)
    return float(val), (_dev.host(grad) if host else grad)


class NetBoxes:
    """First/second extrema per (net, die) with multiplicity (wirelength.py:101-142).
    Attributes cnt/min1/min2/max1/max2 [N,2], full_min/max [N]: CUDA tensors, or
    numpy arrays when the coordinates were given as numpy."""

    def __init__(self, topo, coord, on_top):
        _lib.require_cuda()
        dt = _topo(topo)
        n = dt.n_net
        c = _dev.f64(coord)
        f = _flags(on_top)
        self.cnt = torch.zeros((n, 2), dtype=torch.int64, device="cuda")
        self.min1 = torch.empty((n, 2), dtype=torch.float64, device="cuda")
        self.min2 = torch.empty_like(self.min1)
        self.max1 = torch.empty_like(self.min1)
        self.max2 = torch.empty_like(self.min1)
        self.full_min = torch.empty(n, dtype=torch.float64, device="cuda")
        self.full_max = torch.empty_like(self.full_min)
        self.bistratal = torch.empty_like(self.full_min)
        _lib.call("p3d_netboxes", _lib.byref(dt.struct), _lib.ptr(c), _lib.ptr(f),
                  _lib.ptr(self.cnt), _lib.ptr(self.min1), _lib.ptr(self.min2),
                  _lib.ptr(self.max1), _lib.ptr(self.max2), _lib.ptr(self.full_min),
                  _lib.ptr(self.full_max), _lib.ptr(self.bistratal), _lib.stream_ptr())
        self._dev = {k: getattr(self, k) for k in ("cnt", "min1", "min2", "max1", "max2",
                                                    "full_min", "full_max", "bistratal")}
        # numpy coordinates in (the reference's callers): numpy attributes out
        self._host = isinstance(coord, np.ndarray)
        if self._host:
            for k, v in self._dev.items():
                setattr(self, k, v.cpu().numpy())

    def spans(self):
        """(top span, bottom span, full span); empty partial nets span 0
        (wirelength.py:136-142; p3d_net_spans)."""
        d = [self._dev[k] for k in ("cnt", "min1", "max1", "full_min", "full_max")]
        n = d[0].shape[0]
        top, bot, full = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3))
        _lib.call("p3d_net_spans", int(n), *[_lib.ptr(t) for t in d], _lib.ptr(top),
                  _lib.ptr(bot), _lib.ptr(full), _lib.stream_ptr())
        if self._host:
            return top.cpu().numpy(), bot.cpu().numpy(), full.cpu().numpy()
        return top, bot, full


def bistratal_axis(coords, on_top):
    """Minimal per-axis D2D HPWL of one net (wirelength.py:145-150)."""
    c = np.asarray(coords, dtype=float)
    n = len(c)
    if n == 0:
        return 0.0
    topo = NetTopology(np.array([0, n]), np.zeros(n, np.int64), np.arange(n), n)
    return float(bistratal_spans(topo, c, np.asarray(on_top, bool))[0].item())


def optimal_region(top_box, bot_box):
    """Zero-cost terminal region (wirelength.py:153-164); scalar geometry."""
    out = []
    for a in (0, 2):
        lo = max(top_box[a], bot_box[a])
        hi = min(top_box[a + 1], bot_box[a + 1])
        out.extend((min(lo, hi), max(lo, hi)))
    return tuple(out)


def optimal_hbt_centers(arrays, x, y, z, rot, dz):
    """Optimal-region centre per crossing net (wirelength.py:325-342):
    {net index: (cx, cy)} for nets with pins on both dies.  The per-die boxes
    run on the device (NetBoxes); the region centres are formed vectorised
    with optimal_region's arithmetic ((min(lo, hi) + max(lo, hi)) / 2 ==
    (lo + hi) / 2 exactly) and the dict is assembled once."""
    topo = NetTopology.from_arrays(arrays)
    px, py, _, on_top = dynamic_pin_coords(arrays, x, y, z, rot, dz)
    bx = NetBoxes(topo, px, on_top)
    by = NetBoxes(topo, py, on_top)
    cnt = _dev.host(bx.cnt)
    crossing = np.flatnonzero((cnt[:, 0] > 0) & (cnt[:, 1] > 0))
    mnx, mxx = _dev.host(bx.min1)[crossing], _dev.host(bx.max1)[crossing]
    mny, mxy = _dev.host(by.min1)[crossing], _dev.host(by.max1)[crossing]

    def centre(mn, mx):  # optimal_region on one axis: top box index 1, bottom index 0
        lo = np.maximum(mn[:, 1], mn[:, 0])
        hi = np.minimum(mx[:, 1], mx[:, 0])
        return (np.minimum(lo, hi) + np.maximum(lo, hi)) / 2

    cx, cy = centre(mnx, mxx), centre(mny, mxy)
    return dict(zip(crossing.tolist(), zip(cx.tolist(), cy.tolist())))


@_dev.numpy_io("coord")
def bistratal_spans(topo, coord, on_top, boxes=None):
    """Per-net exact bistratal extent on one axis (wirelength.py:167-170)."""
    if boxes is not None:
        return boxes.bistratal
    return NetBoxes(topo, coord, on_top).bistratal


@_dev.numpy_io("pin_x")
def planar_objective(topo, pin_x, pin_y, on_top, gamma, boxes_x=None, boxes_y=None):
    """Smoothed bistratal WL + per-pin planar gradients (wirelength.py:173-192).
    The branch per net/axis is re-derived on the device from the same exact
    boxes (``boxes_x/boxes_y`` are accepted for signature compatibility)."""
    _lib.require_cuda()
    dt = _topo(topo)
    x, y, f = _dev.f64(pin_x), _dev.f64(pin_y), _flags(on_top)
    gx = torch.empty(dt.n_pin, dtype=torch.float64, device="cuda")
    gy = torch.empty_like(gx)
    val = torch.zeros(1, dtype=torch.float64, device="cuda")
    scr = _dev.scratch(_SCR)
    if dt.n_net:
        _lib.call("p3d_planar_objective_ex", _lib.byref(dt.struct), _lib.ptr(x), _lib.ptr(y),
                  _lib.ptr(f), float(gamma), _lib.ptr(val), _lib.ptr(gx), _lib.ptr(gy),
                  _lib.ptr(scr), _lib.stream_ptr())
    return float(val.item()), gx, gy


@_dev.numpy_io("pin_z")
def z_cut_penalty(topo, pin_z, gamma):
    """Smoothed z-span per net and per-pin gradients (wirelength.py:195-198)."""
    _lib.require_cuda()
    dt = _topo(topo)
    z = _dev.f64(pin_z)
    g = torch.empty(dt.n_pin, dtype=torch.float64, device="cuda")
    val = torch.zeros(1, dtype=torch.float64, device="cuda")
    scr = _dev.scratch(_SCR)
    if dt.n_net:
        _lib.call("p3d_z_cut_penalty_ex", _lib.byref(dt.struct), _lib.ptr(z), float(gamma),
                  _lib.ptr(val), _lib.ptr(g), _lib.ptr(scr), _lib.stream_ptr())
    return float(val.item()), g


def _fd(topo, pin_x, pin_y, on_top, dz, net_has_dup):
    _lib.require_cuda()
    if isinstance(topo, NetTopology):
        dt = DeviceTopology(np.asarray(topo.net_ptr), np.asarray(topo.pin_inst), int(topo.n_obj),
                            net_has_dup)
    else:
        dt = topo
    x, y, f = _dev.f64(pin_x), _dev.f64(pin_y), _flags(on_top)
    g = torch.zeros(max(dt.n_obj, 1), dtype=torch.float64, device="cuda")
    scr = torch.zeros(4 * dt.n_pin + 4 * dt.n_obj + 1, dtype=torch.float64, device="cuda")
    _lib.call("p3d_fd_z_gradient", _lib.byref(dt.struct), _lib.ptr(x), _lib.ptr(y), _lib.ptr(f),
              float(dz), _lib.ptr(g), _lib.ptr(scr), _lib.stream_ptr())
    return g[: dt.n_obj]


@_dev.numpy_io("pin_x")
def fd_z_gradient_incremental(topo, pin_x, pin_y, on_top, dz, net_has_dup=None,
                              boxes_x=None, boxes_y=None):
    """Depth gradient by single-pin die flips (wirelength.py:251-293): O(1) per
    pin from first/second extrema; nets where an owner has several pins take
    the exact per-owner re-evaluation."""
    if net_has_dup is None:
        net_has_dup = net_dup_flags(np.asarray(topo.net_ptr), np.asarray(topo.pin_inst))
    return _fd(topo, pin_x, pin_y, on_top, dz, np.asarray(net_has_dup, bool))


@_dev.numpy_io("pin_x")
def fd_z_gradient_naive(topo, pin_x, pin_y, on_top, dz):
    """Per-owner forced re-evaluation of every net (wirelength.py:205-224):
    the exact O(|P_e|^2) device path applied to all nets."""
    return _fd(topo, pin_x, pin_y, on_top, dz, np.ones(topo.n_net, dtype=bool))


@_dev.numpy_io("grad_x")
def normalize_z_gradient(grad_x, grad_y, grad_z_bistratal, grad_z_hbt, alpha):
    """Eq. 17 (wirelength.py:296-305)."""
    _lib.require_cuda()
    gx, gy = _dev.f64(grad_x), _dev.f64(grad_y)
    gb, gh = _dev.f64(grad_z_bistratal), _dev.f64(grad_z_hbt)
    n = gb.numel()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    scr = _dev.scratch(8 + 3 * 1024)
    _lib.call("p3d_normalize_z_gradient", int(n), _lib.ptr(gx), _lib.ptr(gy), _lib.ptr(gb),
              _lib.ptr(gh), float(alpha), _lib.ptr(out), _lib.ptr(scr), _lib.stream_ptr())
    return out


def rotated_pin_offsets(arrays, rot):
    """[n_pin][4] (rx_top, ry_top, rx_bot, ry_bot), fixed while GP runs."""
    rot = np.asarray(rot)
    if not np.any(rot % 4):  # no quarter turn anywhere (every first GP pass): the offsets
        return np.ascontiguousarray(np.stack([arrays.ox_top, arrays.oy_top, arrays.ox_bot,
                                              arrays.oy_bot], axis=1), dtype=np.float64)
    q = rot[arrays.pin_inst]
    rx_t, ry_t = rotate_offsets(arrays.ox_top, arrays.oy_top, q)
    rx_b, ry_b = rotate_offsets(arrays.ox_bot, arrays.oy_bot, q)
    return np.ascontiguousarray(np.stack([rx_t, ry_t, rx_b, ry_b], axis=1))


@_dev.numpy_io("x")
def dynamic_pin_coords(arrays: NetlistArrays, x, y, z, rot, dz):
    """Absolute pin coordinates with offsets picked by the owner's die
    (wirelength.py:308-322).  Returns CUDA tensors (px, py, pz, on_top bool)."""
    _lib.require_cuda()
    topo = NetTopology.from_arrays(arrays).device(arrays.net_has_dup_inst)
    off = _dev.f64(rotated_pin_offsets(arrays, rot))
    xd, yd, zd = _dev.f64(x), _dev.f64(y), _dev.f64(z)
    n = topo.n_pin
    px = torch.empty(n, dtype=torch.float64, device="cuda")
    py, pz = torch.empty_like(px), torch.empty_like(px)
    top = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.call("p3d_pin_coords", _lib.byref(topo.struct), _lib.ptr(xd), _lib.ptr(yd), _lib.ptr(zd),
              _lib.ptr(off), float(dz), _lib.ptr(px), _lib.ptr(py), _lib.ptr(pz), _lib.ptr(top),
              _lib.stream_ptr())
    return px, py, pz, top.to(torch.bool)


@_dev.numpy_io("x")
def gp_wirelength_objective(arrays, x, y, z, rot, dz, gamma, alpha):
    """Instance-level GP wirelength objective (wirelength.py:345-358): the
    smoothed bistratal total plus alpha times the smoothed z-span total, and
    dW/dx, dW/dy summed per instance.  Pins, both objectives and the
    pin -> instance sums (p3d_gather_pins: per owner in pin order, the
    np.bincount order) all run on the device."""
    _lib.require_cuda()
    topo = NetTopology.from_arrays(arrays)
    dt = topo.device()
    px, py, pz, on_top = dynamic_pin_coords(arrays, _dev.f64(x), _dev.f64(y), _dev.f64(z), rot, dz)
    w_bi, gx_pin, gy_pin = planar_objective(dt, px, py, on_top, gamma)
    w_cut, _ = z_cut_penalty(dt, pz, gamma)
    n_obj = max(int(topo.n_obj), 1)
    pin4 = torch.zeros((max(dt.n_pin, 1), 4), dtype=torch.float64, device="cuda")
    obj4 = torch.zeros(4 * n_obj, dtype=torch.float64, device="cuda")
    if dt.n_pin:
        slot = dt.pin_slot.long()
        pin4[slot, 0] = gx_pin
        pin4[slot, 1] = gy_pin
        _lib.call("p3d_gather_pins", _lib.byref(dt.struct), _lib.ptr(pin4), _lib.ptr(obj4),
                  _lib.stream_ptr())
    n = int(topo.n_obj)
    return w_bi + alpha * w_cut, obj4[:n].clone(), obj4[n_obj: n_obj + n].clone()


__all__ = [
    "optimal_hbt_centers",
    "NetTopology", "DeviceTopology", "partial_hpwl", "wa_smooth", "NetBoxes", "bistratal_axis",
    "optimal_region", "bistratal_spans", "planar_objective", "z_cut_penalty",
    "fd_z_gradient_naive", "fd_z_gradient_incremental", "normalize_z_gradient",
    "dynamic_pin_coords", "rotated_pin_offsets", "partition_from_z", "gp_wirelength_objective",
]
