"""Die utilisation rebalance on the B200 (``place3d.legalize.rebalance_partition``,
legalize.py:464-499).

Same signature and semantics as the reference: moves instances off the die
whose utilisation overshoots its cap more (cells before macros, then the
smallest area on that die, then the lowest index) until both caps hold,
rewriting ``state.z`` of every moved instance to its new die plane; raises
``LegalizationError`` when both caps are exceeded at once or no candidate is
left.  The candidate orders are sorted on the device and one CTA
(``p3d_rebalance``) walks them with block prefix sums (p3d_post.cu); the
decisions equal the reference's whenever the instance areas are integers
(every synthetic / database-unit design), since the area sums are then exact.
The rest of the reference's legalizer stays host code (out of scope).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .model import partition_from_z, rotated_dims


class LegalizationError(RuntimeError):
    """legalize.py:23."""


def _order(area, is_macro):
    """Instance indices sorted by (is_macro, area, index) (legalize.py:493-494)."""
    idx = torch.argsort(area, stable=True)
    idx = idx[torch.argsort(is_macro[idx], stable=True)]
    return idx.to(torch.int32).contiguous()


def rebalance_partition(design, state):
    _lib.require_cuda()
    arr = design.arrays()
    die = design.die
    n = design.n_insts
    delta = partition_from_z(state.z, state.dz).astype(np.uint8)
    wt, ht = rotated_dims(arr.w_top, arr.h_top, state.rot)
    wb, hb = rotated_dims(arr.w_bot, arr.h_bot, state.rot)
    a_top, a_bot = _dev.f64(wt * ht), _dev.f64(wb * hb)
    mac = _dev.u8(arr.is_macro)
    d_delta = _dev.u8(delta)
    out = torch.zeros(4, dtype=torch.float64, device="cuda")
    o_top, o_bot = _order(a_top, mac), _order(a_bot, mac)  # alive until the kernel ran
    _lib.call("p3d_rebalance", int(n), _lib.ptr(a_top), _lib.ptr(a_bot),
              _lib.ptr(o_top), _lib.ptr(o_bot), _lib.ptr(d_delta),
              float(die.max_util_top * die.area), float(die.max_util_bottom * die.area),
              _lib.ptr(out), _lib.stream_ptr())
    status, moves, over_top, over_bot = out.cpu().tolist()
    new = d_delta.cpu().numpy()
    moved = np.flatnonzero(new & 2)  # moved at least once: z on its final die's plane
    state.z[moved] = np.where((new[moved] & 1) == 1, 3 * state.dz / 4, state.dz / 4)
    if status == 1:
        raise LegalizationError(f"utilization caps unsatisfiable (top over {over_top:.0f},"
                                f" bottom over {over_bot:.0f})")
    if status == 2:
        raise LegalizationError("utilization rebalancing did not converge")
    return state


__all__ = ["LegalizationError", "rebalance_partition"]
