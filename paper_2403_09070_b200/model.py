"""Host-side design container for the GP hot path.

The reference keeps a fully cross-linked ``Design`` (``place3d/model.py:119-221``)
and derives flat numeric views from it (``NetlistArrays``, ``model.py:224-275``).
The GP loop only ever touches those flat views plus a handful of scalars
(die extents, row heights, utilisation caps, HBT pitch/cost).  This module holds
exactly that: ``ArrayDesign`` is a duck-type of the reference ``Design`` as far
as ``run_gp3d`` / ``Gp3dProblem`` are concerned, so either object can be
handed to :mod:`paper_2403_09070_b200.gp`.

Conventions follow the reference: instance centre coordinates, die 0 = bottom,
die 1 = top, pins in CSR order by net.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class DieSpec:
    """Mirror of ``place3d.model.DieSpec`` (``model.py:77-94``)."""

    width: float
    height: float
    row_height_top: float
    row_height_bottom: float
    max_util_top: float
    max_util_bottom: float
    site_width: float = 1.0

    @property
    def area(self):
        return self.width * self.height


@dataclass(frozen=True)
class HbtSpec:
    """Mirror of ``place3d.model.HbtSpec`` (``model.py:97-101``)."""

    pitch: float
    spacing: float
    cost: float


class NetlistArrays:
    """Flat CSR netlist (same attribute names as ``model.py:224-275``).

    Built from already-flat arrays; ``pin_degree`` and ``net_has_dup_inst`` are
    derived exactly as the reference derives them (``model.py:267-275``).
    """

    def __init__(self, *, is_macro, w_top, h_top, w_bot, h_bot, net_ptr, pin_inst,
                 ox_top, oy_top, ox_bot, oy_bot):
        self.is_macro = np.asarray(is_macro, dtype=bool)
        self.n_inst = len(self.is_macro)
        self.w_top = np.asarray(w_top, dtype=np.float64)
        self.h_top = np.asarray(h_top, dtype=np.float64)
        self.w_bot = np.asarray(w_bot, dtype=np.float64)
        self.h_bot = np.asarray(h_bot, dtype=np.float64)
        self.net_ptr = np.asarray(net_ptr, dtype=np.int64)
        self.n_net = len(self.net_ptr) - 1
        self.pin_inst = np.asarray(pin_inst, dtype=np.int64)
        self.n_pin = len(self.pin_inst)
        self.pin_net = np.repeat(np.arange(self.n_net, dtype=np.int64),
                                 np.diff(self.net_ptr))
        self.ox_top = np.asarray(ox_top, dtype=np.float64)
        self.oy_top = np.asarray(oy_top, dtype=np.float64)
        self.ox_bot = np.asarray(ox_bot, dtype=np.float64)
        self.oy_bot = np.asarray(oy_bot, dtype=np.float64)
        self.pin_degree = np.bincount(self.pin_inst, minlength=self.n_inst).astype(np.int64)
        self.net_has_dup_inst = net_dup_flags(self.net_ptr, self.pin_inst)


def net_dup_flags(net_ptr, pin_inst):
    """True for nets in which one instance owns two or more pins
    (the reference's ``net_has_dup_inst``, ``model.py:268-275``)."""
    net_ptr = np.asarray(net_ptr, dtype=np.int64)
    n_net = len(net_ptr) - 1
    pin_net = np.repeat(np.arange(n_net, dtype=np.int64), np.diff(net_ptr))
    flags = np.zeros(n_net, dtype=bool)
    if len(pin_inst) > 1:
        key = np.lexsort((np.asarray(pin_inst), pin_net))
        sn, si = pin_net[key], np.asarray(pin_inst)[key]
        rep = (sn[1:] == sn[:-1]) & (si[1:] == si[:-1])
        flags[sn[1:][rep]] = True
    return flags


class ArrayDesign:
    """The subset of ``place3d.model.Design`` the GP loop reads."""

    def __init__(self, die: DieSpec, hbt: HbtSpec, arrays: NetlistArrays, name="design"):
        self.die = die
        self.hbt = hbt
        self._arrays = arrays
        self.name = name

    @property
    def n_insts(self):
        return self._arrays.n_inst

    @property
    def n_nets(self):
        return self._arrays.n_net

    @property
    def r_ma(self):
        a = self._arrays
        return float((a.w_bot[a.is_macro] * a.h_bot[a.is_macro]).sum() / self.die.area)

    def arrays(self):
        return self._arrays


@dataclass
class PlacementState:
    """Mirror of ``place3d.model.PlacementState`` (``model.py:298-313``)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    rot: np.ndarray
    dz: float
    fillers: object = None

    def copy(self):
        return PlacementState(self.x.copy(), self.y.copy(), self.z.copy(),
                              self.rot.copy(), self.dz, self.fillers)


def partition_from_z(z, dz):
    """delta = 1 iff z - dz/2 > 0 (``model.py:316-318``; the midplane is die 0)."""
    return (np.asarray(z) - dz / 2 > 0).astype(np.int8)


def rotate_offsets(ox, oy, quarters):
    """Quarter-turn CCW rotation of pin offsets (``model.py:278-289``)."""
    q = np.asarray(quarters) % 4
    ox = np.asarray(ox, dtype=np.float64)
    oy = np.asarray(oy, dtype=np.float64)
    rx = np.choose(q, [ox, -oy, -ox, oy])
    ry = np.choose(q, [oy, ox, -oy, -ox])
    return rx, ry


def rotated_dims(w, h, quarters):
    """Swap footprint sides on odd quarter turns (``model.py:292-295``)."""
    odd = (np.asarray(quarters) % 4) % 2 == 1
    return np.where(odd, h, w), np.where(odd, w, h)


class ParseError(ValueError):
    """Malformed design text (model.py:28-35); the message carries the line."""


def parse_design_arrays(stream) -> ArrayDesign:
    """The reference's ``parse_design`` (model.py:423-571) with its Design
    checks (model.py:121-190), straight to the flat arrays the GP loop reads
    (``NetlistArrays``, model.py:231-275): one native pass over the text
    (``p3d_parse_design``, host C++) instead of Python objects per instance
    and pin.  ``stream``: the text, or an iterable of lines / a file object.
    Raises ``ParseError`` with the reference's message on malformed input.
    Instance / net names are kept (``inst_names``, ``net_names``) for the
    solution check's messages."""
    import ctypes as C

    from . import _lib

    if isinstance(stream, bytes):
        text = stream
    elif isinstance(stream, str):
        text = stream.encode()
    else:
        text = "".join(stream).encode()
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.p3d_parse_design(text, len(text), C.byref(h))
    if rc != 0:
        buf = C.create_string_buffer(1024)
        lib.p3d_last_error(buf, 1024)
        raise ParseError(buf.value.decode(errors="replace"))
    try:
        counts = np.zeros(5, dtype=np.int64)
        sc = np.zeros(9)
        lib.p3d_parsed_counts(h, counts.ctypes.data, sc.ctypes.data)
        n, m, p, ib, nb = (int(v) for v in counts)
        is_macro = np.zeros(n, dtype=np.uint8)
        wt, ht, wb, hb = (np.zeros(n) for _ in range(4))
        net_ptr = np.zeros(m + 1, dtype=np.int64)
        pin_inst = np.zeros(p, dtype=np.int64)
        oxt, oyt, oxb, oyb = (np.zeros(p) for _ in range(4))
        inames, nnames = C.create_string_buffer(max(ib, 1)), C.create_string_buffer(max(nb, 1))
        lib.p3d_parsed_fill(h, *(a.ctypes.data for a in (is_macro, wt, ht, wb, hb, net_ptr,
                                                         pin_inst, oxt, oyt, oxb, oyb)),
                            inames, nnames)
    finally:
        lib.p3d_parsed_free(h)
    arr = NetlistArrays(is_macro=is_macro.astype(bool), w_top=wt, h_top=ht, w_bot=wb, h_bot=hb,
                        net_ptr=net_ptr, pin_inst=pin_inst, ox_top=oxt, oy_top=oyt, ox_bot=oxb,
                        oy_bot=oyb)
    sc = [float(v) for v in sc]
    die = DieSpec(width=sc[0], height=sc[1], row_height_top=sc[2], row_height_bottom=sc[3],
                  max_util_top=sc[4], max_util_bottom=sc[5])
    d = ArrayDesign(die, HbtSpec(sc[6], sc[7], sc[8]), arr)
    d.inst_names = inames.raw[:ib].decode().split("\n")[:n]
    d.net_names = nnames.raw[:nb].decode().split("\n")[:m]
    return d
