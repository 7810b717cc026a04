"""The reference's own unit tests for the host-side pieces of the GP path,
restated against this package (no reference import): the loop-control
scalars of gp.py (lambda init, mu rule, gamma schedule, flow selection,
alpha), the optimal region, the corner stamp, the filler builder and the
field dump.  Each test cites the reference test it restates
(pkg/tests/<file>:<line>).  The device-side tests of the same files are in
test_gpu_reference_suite.py.  Runs on CPU."""

import math

import numpy as np
import pytest

from paper_2403_09070_b200 import density as dn
from paper_2403_09070_b200 import gp as gpm
from paper_2403_09070_b200 import wirelength as wl
from refsuite import make_design, make_kind


# -- test_gp.py ----------------------------------------------------------------


def test_lambda_init_guards():
    """test_gp.py:37."""
    assert gpm.lambda_init(0.0, 5.0) == 1e-3
    assert gpm.lambda_init(5.0, 0.0) == 1e-3
    assert gpm.lambda_init(7.0, 7.0) == pytest.approx(1e-3)
    assert gpm.lambda_init(14.0, 7.0) == pytest.approx(2e-3)


def test_mu_compound_growth():
    """test_gp.py:44."""
    lam = 1.0
    for _ in range(100):
        lam *= 1.02
    assert lam == pytest.approx(1.02 ** 100) and lam == pytest.approx(7.2446, rel=1e-4)


def test_mu_respects_bounds():
    """test_gp.py:52."""
    cfg = gpm.GpConfig()
    for prev, cur in ((1.0, 0.5), (0.5, 0.4999), (0.5, 0.5), (math.inf, 1.0)):
        assert cfg.mu_min <= gpm.mu_from_overflow(prev, cur, cfg) <= cfg.mu_max


def _two_inst(km, die):
    k = make_kind("c", 2, 2, [("p", 0, 0)])
    return make_design([k, km], [k, km], [("a", "c", False), ("m0", "m", True)],
                       [("n", [(0, "p"), (1, "p")])], die=die, rows=(2, 2))


def test_select_flow_thresholds():
    """test_gp.py:59: bottom-die macro area 60*58 over 100*96 = 0.3625 -> 3d;
    96*88 over 9600 > 0.5 -> 2d."""
    assert gpm.select_flow(_two_inst(make_kind("m", 60, 58, [("p", 0, 0)]), (100, 96))) == "3d"
    d2 = _two_inst(make_kind("m", 96, 88, [("p", 0, 0)]), (100, 96))
    assert d2.r_ma > 0.5 and gpm.select_flow(d2) == "2d"


def test_select_flow_boundary_inclusive():
    """test_gp.py:77."""
    d = _two_inst(make_kind("m", 96, 50, [("p", 0, 0)]), (96, 100))
    assert d.r_ma == pytest.approx(0.5) and gpm.select_flow(d) == "2d"


def test_alpha_published_fit_dominates_at_scale():
    """test_gp.py:88."""
    k = make_kind("c", 2, 33, [("p", 0, 0)])
    d = make_design([k], [k], [("a", "c", False)], [], die=(52800, 52800), rows=(33, 48),
                    hbt=(92, 10, 10.0))
    dz = 8 * (52800 / 512)
    eta = 2 * 92 / (33 + 48)
    want = 3.5e-3 * (52800 * eta ** 2 / dz) * math.log(90 * 10 * eta - 1)
    assert gpm.alpha_value(d, dz, gpm.GpConfig()) == pytest.approx(want)


def test_alpha_guard_clamps_log_argument():
    """test_gp.py:100."""
    k = make_kind("c", 2, 33, [("p", 0, 0)])
    d = make_design([k], [k], [("a", "c", False)], [], die=(528, 528), rows=(33, 48),
                    hbt=(1, 0, 0.0))
    assert gpm.alpha_value(d, 100.0, gpm.GpConfig()) >= 0.0


def test_gamma_schedule_endpoints():
    """test_gp.py:276."""
    grid = type("G", (), {"db": 2.0})()
    cfg = gpm.GpConfig()
    assert gpm.gamma_schedule(grid, 0, 100, cfg) == pytest.approx(8.0)
    assert gpm.gamma_schedule(grid, 99, 100, cfg) == pytest.approx(1.0)
    assert 1.0 < gpm.gamma_schedule(grid, 50, 100, cfg) < 8.0


# -- test_wirelength.py: optimal region ------------------------------------------


def test_optimal_region_cases():
    """test_wirelength.py:77, :82, :87."""
    assert wl.optimal_region((0, 2, 0, 2), (1, 3, 1, 3)) == (1, 2, 1, 2)
    assert wl.optimal_region((0, 2, 1, 5), (0, 2, 1, 5)) == (0, 2, 1, 5)
    assert wl.optimal_region((0, 1, 0, 1), (2, 3, 2, 3)) == (1, 2, 1, 2)


def test_optimal_region_touches_both_hulls():
    """test_wirelength.py:92."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        t = np.sort(rng.integers(0, 50, 4))
        b = np.sort(rng.integers(0, 50, 4))
        top, bot = tuple(t), tuple(b)
        r = wl.optimal_region(top, bot)
        assert min(top[1], bot[1]) <= r[1] + 1e-9 and r[0] <= max(top[0], bot[0]) + 1e-9
        assert r[0] <= r[1] and r[2] <= r[3]


# -- test_density.py: host helpers ---------------------------------------------------


def test_corner_map_cases():
    """test_density.py:126, :133, :140."""
    grid = dn.DensityGrid(4, 4, 4, 4, 4)
    idx, vals = dn.corner_map((2.0, 3.0, 1.0), grid)
    assert idx == [(2, 3, 1)] and vals == [1.0]
    idx, vals = dn.corner_map((0.5, 0.0, 0.0), grid)
    assert dict(zip(idx, vals)) == {(0, 0, 0): 0.5, (1, 0, 0): 0.5}
    idx, vals = dn.corner_map((0.5, 0.5, 0.5), grid)
    assert len(idx) == 8 and all(v == pytest.approx(0.125) for v in vals)


def test_filler_volumes_exact():
    """test_density.py:458."""
    fs = dn.build_fillers((100.0, 80.0), 16.0, 0.8, 0.7, 25.0, np.random.default_rng(18))
    assert fs.total_volume(1) == pytest.approx(0.5 * 100 * 80 * 16 * (1 - 0.8), rel=1e-12)
    assert fs.total_volume(0) == pytest.approx(0.5 * 100 * 80 * 16 * (1 - 0.7), rel=1e-12)
    assert (fs.z[fs.die == 1] == 12.0).all() and (fs.z[fs.die == 0] == 4.0).all()


def test_dump_and_load_fields(tmp_path):
    """test_density.py:469."""
    grid = dn.DensityGrid(4, 4, 4, 4, 4)
    rho = np.arange(64, dtype=float).reshape(grid.shape)
    paths = dn.dump_fields(str(tmp_path / "f."), grid, {"rho": rho})
    name, back = dn.load_field(paths[0])
    assert name == "rho" and np.array_equal(back, rho)
