"""Independent solution check on the B200 (``place3d.check.check_solution``,
check.py:74-152).

Same signature, report and messages as the reference: per-instance rotation /
die bounds / row and site grid, same-die overlaps, per-die utilisation, one
terminal per crossing net and none elsewhere, terminal bounds and spacing,
and the score recomputed from scratch (``evaluate_score``, p3d_score).  The
per-object tests and the two pair searches (instance outlines per die,
terminal boxes) run on the device (``p3d_check_objects``, ``p3d_pair_search``:
a uniform bucket grid, every pair reported once); the host only formats the
flagged items' messages from the caller's own solution values, in the
reference's order (overlap and spacing pairs sorted by index, where the
reference follows its hash-bucket order).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .score import evaluate_score


@dataclass
class Violation:
    kind: str
    message: str

    def __str__(self):
        return f"[{self.kind}] {self.message}"


@dataclass
class CheckReport:
    violations: list = field(default_factory=list)
    hpwl: float = 0.0
    hbt_count: int = 0
    raw_score: float = 0.0

    @property
    def passed(self):
        return not self.violations

    def as_dict(self):
        return {"passed": self.passed, "violations": [str(v) for v in self.violations],
                "hpwl": self.hpwl, "hbt_count": self.hbt_count, "raw_score": self.raw_score}


def _names(design):
    """Instance and net names: the design's own, else the synthetic
    generator's convention (cells c<i>, macros m<k>, nets n<j>; synth.py:135-167)."""
    if hasattr(design, "insts") and hasattr(design, "nets"):
        return [x.name for x in design.insts], [e.name for e in design.nets]
    if getattr(design, "inst_names", None) is not None:  # model.parse_design_arrays
        return design.inst_names, design.net_names
    a = design.arrays()
    k = np.cumsum(a.is_macro) - 1
    inst = [f"m{k[i]}" if a.is_macro[i] else f"c{i}" for i in range(design.n_insts)]
    return inst, [f"n{j}" for j in range(design.n_nets)]


def _pairs(box, member, bucket, extent_x, extent_y, mode=0, min_cc=0.0, tol=0.0):
    """Every pair (p < q) of member boxes the device pair search reports."""
    n = int(member.numel())
    if n == 0 or int(member.sum().item()) < 2:
        return np.zeros((0, 2), dtype=np.int64)
    nbx = max(1, int(np.ceil(extent_x / bucket)) + 1)
    nby = max(1, int(np.ceil(extent_y / bucket)) + 1)
    count = torch.zeros(nbx * nby, dtype=torch.int32, device="cuda")
    s = _lib.stream_ptr()
    args = lambda ph, start, cursor, lst, out, cap, n_out: (  # noqa: E731
        ph, n, _lib.ptr(box), _lib.ptr(member), float(bucket), nbx, nby, mode, float(min_cc),
        float(tol), _lib.ptr(count), start, cursor, lst, out, cap, n_out, s)
    _lib.call("p3d_pair_search", *args(0, None, None, None, None, 0, None))
    start = torch.zeros(nbx * nby + 1, dtype=torch.int32, device="cuda")
    start[1:] = torch.cumsum(count, 0)
    total = int(start[-1].item())
    cursor = start[:-1].clone()
    lst = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    _lib.call("p3d_pair_search", *args(1, None, _lib.ptr(cursor), _lib.ptr(lst), None, 0, None))
    cap = 1 << 16
    while True:
        out = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
        n_out = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("p3d_pair_search", *args(2, _lib.ptr(start), None, _lib.ptr(lst), _lib.ptr(out),
                                           cap, _lib.ptr(n_out)))
        k = int(n_out.item())
        if k <= cap:
            res = out[:k].cpu().numpy().astype(np.int64)
            return res[np.lexsort((res[:, 1], res[:, 0]))] if k else res
        cap = k


def check_solution(design, sol, tol=1e-6):
    _lib.require_cuda()
    rep = CheckReport()
    bad = rep.violations.append
    die = design.die
    a = design.arrays()
    n, n_net = design.n_insts, design.n_nets
    inst_name, net_name = _names(design)
    s_die = np.asarray(sol.die).astype(np.int64)
    s_rot = np.asarray(sol.rot).astype(np.int64)
    s_x = np.asarray(sol.x, dtype=np.float64)
    s_y = np.asarray(sol.y, dtype=np.float64)
    ok = np.zeros(max(n_net, 1), dtype=bool)
    hx, hy = np.zeros(max(n_net, 1)), np.zeros(max(n_net, 1))
    for j, (x, y) in sol.hbt_xy.items():
        ok[int(j)] = True
        hx[int(j)], hy[int(j)] = float(x), float(y)
    inst_flags = torch.zeros(n, dtype=torch.uint8, device="cuda")
    net_flags = torch.zeros(max(n_net, 1), dtype=torch.uint8, device="cuda")
    box = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    area = torch.zeros(2, dtype=torch.float64, device="cuda")
    scr = _dev.scratch(8 + 2 * 2048)
    t = [_dev.u8(s_die == 1), _dev.i32(s_rot), _dev.f64(s_x), _dev.f64(s_y), _dev.u8(a.is_macro),
         _dev.f64(a.w_top), _dev.f64(a.h_top), _dev.f64(a.w_bot), _dev.f64(a.h_bot),
         _dev.i32(a.net_ptr), _dev.i32(a.pin_inst if len(a.pin_inst) else np.zeros(1, np.int64)),
         _dev.u8(ok), _dev.f64(hx), _dev.f64(hy)]
    _lib.call("p3d_check_objects", int(n), int(n_net), *[_lib.ptr(v) for v in t],
              float(die.width), float(die.height), float(die.row_height_top),
              float(die.row_height_bottom), float(die.site_width), float(design.hbt.pitch),
              float(tol), _lib.ptr(inst_flags), _lib.ptr(net_flags), _lib.ptr(box),
              _lib.ptr(area), _lib.ptr(scr), _lib.stream_ptr())
    fl = inst_flags.cpu().numpy()
    # per instance, in index order (check.py:78-101)
    for i in np.flatnonzero(fl):
        f = int(fl[i])
        d = int(s_die[i])
        q = int(s_rot[i]) % 4
        x0, y0 = float(sol.x[i]), float(sol.y[i])
        if f & 1:
            bad(Violation("rotation", f"cell {inst_name[i]} rotated {q * 90} deg"))
        if f & 2:
            bad(Violation("bounds", f"{inst_name[i]} at ({x0},{y0}) leaves the die"))
        if f & 4:
            rh = die.row_height_top if d == 1 else die.row_height_bottom
            bad(Violation("row", f"cell {inst_name[i]} y={y0} off the row grid ({rh})"))
        if f & 8:
            bad(Violation("site", f"cell {inst_name[i]} x={x0} off the site grid"))
    # same-die overlaps (check.py:103-110)
    bucket = max(die.width, die.height) / 32
    bx = box.cpu().numpy()
    d_die = _dev.u8(s_die == 1)
    for d in (0, 1):
        member = d_die if d == 1 else (1 - d_die)
        for p, q in _pairs(box, member.contiguous(), bucket, die.width, die.height):
            bad(Violation("overlap", f"die {d}: {inst_name[p]} ({float(bx[p, 0])},{float(bx[p, 2])}) overlaps "
                                     f"{inst_name[q]} ({float(bx[q, 0])},{float(bx[q, 2])})"))
    # utilisation (check.py:112-118)
    ar = area.cpu().tolist()
    for d in (0, 1):
        cap = (die.max_util_top if d == 1 else die.max_util_bottom) * die.area
        if ar[d] > cap * (1 + 1e-9) + tol:
            bad(Violation("utilization", f"die {d}: area {ar[d]:.0f} exceeds cap {cap:.0f}"))
    # terminals (check.py:120-139)
    nf = net_flags.cpu().numpy()[:n_net]
    for j in np.flatnonzero(nf & 3):
        if nf[j] & 1:
            bad(Violation("hbt", f"crossing net {net_name[j]} has no terminal"))
        else:
            bad(Violation("hbt", f"single-die net {net_name[j]} carries a terminal"))
    pitch = design.hbt.pitch
    min_cc = pitch + design.hbt.spacing
    for j, _ in sorted(sol.hbt_xy.items()):
        if nf[int(j)] & 4:
            bad(Violation("hbt-bounds", f"terminal of {net_name[int(j)]} leaves the die"))
    keys = sorted(int(j) for j in sol.hbt_xy)
    if len(keys) > 1:
        kx = np.array([float(sol.hbt_xy[j][0]) for j in keys])
        ky = np.array([float(sol.hbt_xy[j][1]) for j in keys])
        hbox = _dev.f64(np.c_[kx, kx + min_cc, ky, ky + min_cc])
        member = torch.ones(len(keys), dtype=torch.uint8, device="cuda")
        hb = max(min_cc * 4, 1.0)
        ext_x = max(die.width, float(kx.max()) + min_cc) + hb
        ext_y = max(die.height, float(ky.max()) + min_cc) + hb
        for p, q in _pairs(hbox, member, hb, ext_x, ext_y, mode=1, min_cc=min_cc, tol=tol):
            j1, j2 = keys[p], keys[q]
            c1, c2 = sol.hbt_xy[j1], sol.hbt_xy[j2]
            sp = max(abs(c1[0] - c2[0]), abs(c1[1] - c2[1]))
            bad(Violation("hbt-spacing", f"terminals of {net_name[j1]} and {net_name[j2]}"
                                         f" spaced {sp} < {min_cc}"))
    score = evaluate_score(design, sol, allow_illegal=True)
    rep.hpwl = score.hpwl
    rep.hbt_count = score.hbt_count
    rep.raw_score = score.raw_score
    return rep


__all__ = ["CheckReport", "Violation", "check_solution"]
