"""CPU checks of the arithmetic identities the kernels rely on to stay
bit-identical to the reference's formulas (exact rational arithmetic where an
FMA is involved).  Each test names the device code it backs."""

from fractions import Fraction

import numpy as np


def _rn(fr):
    return float(fr)  # int / int true division: correctly rounded


def _fma(a, b, c):
    return _rn(Fraction(a) * Fraction(b) + Fraction(c))


def test_shared_reciprocal_quotient_is_the_ieee_quotient():
    """p3d_common.cuh div_rcp: q = x y, q + (x - q b) y with y = RN(1/b)
    equals RN(x / b) (K4 / K5 quotients, footprint bin indices)."""
    rng = np.random.default_rng(11)
    for _ in range(20000):
        x = float(rng.standard_normal() * 10.0 ** rng.integers(-12, 12))
        b = float(abs(rng.standard_normal()) * 10.0 ** rng.integers(-4, 6) + 1e-3)
        y = 1.0 / b
        q = x * y
        got = _fma(_fma(-q, b, x), y, q)
        assert got == _rn(Fraction(x) / Fraction(b)), (x, b)


def test_branch_free_top2_equals_the_if_chain():
    """p3d_wl_fused.cu Side::push: hi2' = max(hi2, min(hi1, h)), hi1' =
    max(hi1, h) (and the mirrored lo update) keep exactly the values of the
    if / else-if chain, ties and -inf sentinels included."""
    rng = np.random.default_rng(5)
    for _ in range(3000):
        vals = list(rng.integers(0, 6, size=rng.integers(1, 8)).astype(float))
        hi1 = hi2 = -np.inf
        lo1 = lo2 = np.inf
        h1 = h2 = -np.inf
        l1 = l2 = np.inf
        for c in vals:
            if c > hi1:
                hi2, hi1 = hi1, c
            elif c > hi2:
                hi2 = c
            if c < lo1:
                lo2, lo1 = lo1, c
            elif c < lo2:
                lo2 = c
            h2 = max(h2, min(h1, c))
            h1 = max(h1, c)
            l2 = min(l2, max(l1, c))
            l1 = min(l1, c)
            # a neutral push leaves the other side unchanged
            h2n, h1n = max(h2, min(h1, -np.inf)), max(h1, -np.inf)
            assert (h2n, h1n) == (h2, h1)
        assert (h1, h2, l1, l2) == (hi1, hi2, lo1, lo2)


def _overlap_len(lo, hi, i, step):
    return max(min(hi, (i + 1) * step) - max(lo, i * step), 0.0)


def _axis_span(c, size, extent, step, n):
    lo = min(max(c - size / 2, 0.0), extent)
    hi = min(max(c + size / 2, 0.0), extent)
    a = int(np.floor(lo / step))
    b = int(np.ceil(hi / step)) - 1
    a = min(max(a, 0), n - 1)
    b = min(max(b, 0), n - 1)
    return lo, hi, a, max(a, b)


def _axis_weights(lo, hi, i0, i1, step, m):
    """p3d_geom.cuh axis_weights: interior boundaries without min / max."""
    nr = i1 - i0 + 1
    e = [(float(i0) + k) * step for k in range(m + 1)]
    right_edge = e[m]
    for k in range(1, m):
        if nr == k:
            right_edge = e[k]
    right_edge = min(hi, right_edge)
    w = []
    for k in range(m):
        right = right_edge if k == nr - 1 else e[k + 1]
        v = max(right - max(lo, e[0]), 0.0) if k == 0 else right - e[k]
        w.append(v if k < nr else 0.0)
    return w


def test_axis_weights_equal_overlap_len():
    """The footprint weights of K2 / K4 equal density.py's per-bin overlap
    lengths bit for bit (density.py:172-173), edges and clipping included."""
    rng = np.random.default_rng(3)
    for _ in range(20000):
        n = int(rng.integers(2, 600))
        step = float(rng.uniform(0.5, 80.0))
        extent = n * step
        size = float(rng.uniform(0.0, 2.9 * step))
        c = float(rng.uniform(-step, extent + step))
        if rng.random() < 0.1:  # centres on bin boundaries
            c = float(rng.integers(0, n + 1)) * step + (size / 2 if rng.random() < 0.5 else 0.0)
        lo, hi, i0, i1 = _axis_span(c, size, extent, step, n)
        if i1 - i0 + 1 > 3:
            continue
        got = _axis_weights(lo, hi, i0, i1, step, 3)
        want = [_overlap_len(lo, hi, i0 + k, step) if k <= i1 - i0 else 0.0 for k in range(3)]
        assert got == want, (c, size, step, n)


def test_degree3_nets_are_never_split_and_have_zero_flip_delta():
    """p3d_wl_fused.cu triple_task: for 3 pins on two dies, top + bottom span
    <= full span, and every flip delta max(full, sp + op) - full is 0
    (wirelength.py:186, 227-248)."""
    rng = np.random.default_rng(9)
    for _ in range(5000):
        v = rng.uniform(0, 100, 3).round(rng.integers(0, 3))
        d = rng.integers(0, 2, 3)
        full = v.max() - v.min()
        spans = [(v[d == s].max() - v[d == s].min()) if (d == s).sum() > 0 else 0.0 for s in (0, 1)]
        assert spans[0] + spans[1] <= full
        for k in range(3):
            same = [v[j] for j in range(3) if j != k and d[j] == d[k]]
            other = [v[j] for j in range(3) if d[j] != d[k]] + [v[k]]
            sp = (max(same) - min(same)) if len(same) > 1 else 0.0
            op = max(other) - min(other)
            assert max(full, sp + op) - full == 0.0
