"""Solution score on the device (evaluate_score, model.py:364-400; SURVEY 8f
rank 4): die-to-die HPWL of a placed solution + HBT cost * #HBTs.

Same signature and result as the reference: ``evaluate_score(design, sol,
allow_illegal=False) -> Score``; ``sol`` carries ``die``, lower-left ``x``/``y``,
``rot`` and ``hbt_xy`` {net: lower-left corner}.  Net-parallel kernel
``p3d_score``; a crossing net without an HBT (or an HBT on a single-die net)
raises ``SolutionError`` unless ``allow_illegal``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib


class SolutionError(ValueError):
    """Solution inconsistent with its design (model.py:43-44)."""


@dataclass
class Score:
    hpwl: float
    hbt_count: int
    raw_score: float


def evaluate_score(design, sol, *, allow_illegal=False):
    _lib.require_cuda()
    a = design.arrays()
    n_net = a.n_net
    ok = np.zeros(n_net, dtype=bool)
    hx = np.zeros(n_net)
    hy = np.zeros(n_net)
    for j, (x, y) in sol.hbt_xy.items():
        ok[int(j)] = True
        hx[int(j)], hy[int(j)] = x, y
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    scr = _dev.scratch(8 + 2 * 1024)
    t = [_dev.i32(a.net_ptr), _dev.i32(a.pin_inst if len(a.pin_inst) else np.zeros(1, np.int64))]
    t += [_dev.f64(v if len(v) else np.zeros(1)) for v in (a.ox_top, a.oy_top, a.ox_bot, a.oy_bot)]
    t += [_dev.f64(v) for v in (a.w_top, a.h_top, a.w_bot, a.h_bot)]
    t += [_dev.u8(np.asarray(sol.die) == 1), _dev.i32(np.asarray(sol.rot) % 4),
          _dev.f64(sol.x), _dev.f64(sol.y), _dev.u8(ok), _dev.f64(hx), _dev.f64(hy)]
    _lib.call("p3d_score", int(n_net), *[_lib.ptr(v) for v in t], float(design.hbt.pitch),
              float(design.hbt.cost), _lib.ptr(out), _lib.ptr(bad), _lib.ptr(scr),
              _lib.stream_ptr())
    if not allow_illegal and int(bad.item()):
        raise SolutionError(f"{int(bad.item())} nets: crossing without an HBT or an HBT on a "
                            "single-die net")
    h, c, r = out.cpu().tolist()
    return Score(hpwl=h, hbt_count=int(c), raw_score=r)


__all__ = ["Score", "SolutionError", "evaluate_score"]
