"""Bit-exact int64 fixed-point density restatement (TEST INFRASTRUCTURE ONLY).

The GPU accumulates rho as int64 in units of 2^-40 per unit density so that
the map is exact and independent of atomic order and GPU count (SURVEY.md
section 0 item 5, Appendix A.4).  The contract, mirrored here:

* every object (cell, filler and macro alike) contributes one term per
  overlapped bin, generated exactly like the reference's direct traversal
  (``density.py:155-196``): clipped box, ``floor``/``ceil`` bin ranges, per-axis
  overlap ``clip(min(hi,(i+1)s) - max(lo,i s), 0)``, volume ``(wx*wy)*wz``;
* the term is ``rint((weight * volume) * fx_scale)`` with
  ``fx_scale = 2**40 / bin_vol`` computed once in float64 (round half to even,
  the same as CUDA ``__double2ll_rn``);
* rho = sum of terms * 2**-40.

Macros therefore use direct per-bin overlap (the GPU's per-macro tile path)
instead of the reference's corner stamps + prefix sum (``density.py:243-298``);
both equal the exact overlap integral, they differ only in fp rounding
(~1e-13 relative, checked against the reference in ``tests/test_oracle.py``).
"""

from __future__ import annotations

import numpy as np

from .port import overlap_terms

FX_BITS = 40


def fx_scale(grid):
    return np.ldexp(1.0, FX_BITS) / grid.bin_vol


def fixed_rho(grid, cl):
    """int64 map [nx, ny, nz] in units of 2^-40."""
    acc = np.zeros(grid.nx * grid.ny * grid.nz, dtype=np.int64)
    s = fx_scale(grid)
    for part in (~cl.is_macro, cl.is_macro):
        if not part.any():
            continue
        sub = cl.take(part)
        for flat, vol in overlap_terms(grid, sub):
            q = np.rint((sub.weight * vol) * s).astype(np.int64)
            nz = q != 0
            np.add.at(acc, flat[nz], q[nz])
    return acc.reshape(grid.shape)


def to_density(acc):
    return acc.astype(np.float64) * np.ldexp(1.0, -FX_BITS)


def fixed_overflow(acc, grid, rho_t, mv):
    """Overflow from the fixed-point map: exact integer excess, one rounding."""
    if mv <= 0:
        return 0.0
    t = np.int64(np.rint(rho_t * np.ldexp(1.0, FX_BITS)))
    ex = int(np.maximum(acc.astype(np.int64) - t, 0).sum())
    return float(ex) * np.ldexp(1.0, -FX_BITS) * grid.bin_vol / mv
