"""The reference's own unit tests for the GP path (pkg/tests/test_wirelength.py,
test_density.py, test_gp.py), restated against the device implementation:
every operator these tests touch runs in libp3d.so and is called with numpy
inputs, as the reference's callers call it, so the tests also pin the
numpy-in / numpy-out drop-in convention.  Same inputs, seeds, assertions and
tolerances as the reference test each one cites (file:line); where the device
arithmetic differs by construction (the int64 fixed-point density map,
2^-40 per unit density) the reference's tolerance already covers it.  The
host-side tests of the same files are in test_reference_suite_host.py."""

import math

import numpy as np
import pytest
from scipy import fft as sfft

from paper_2403_09070_b200 import density as dn
from paper_2403_09070_b200 import gp as gpm
from paper_2403_09070_b200 import wirelength as wl
from paper_2403_09070_b200.model import PlacementState, partition_from_z
from paper_2403_09070_b200.synth import SynthSpec, synth_arrays
from refsuite import brute_density, make_cloud, make_design, make_kind, make_topo, random_net

pytestmark = pytest.mark.gpu


# ==== test_wirelength.py ==========================================================


def test_partial_hpwl():
    """test_wirelength.py:23."""
    assert wl.partial_hpwl([5]) == 0
    assert wl.partial_hpwl([0, 10]) == 10
    assert wl.partial_hpwl([]) == 0


def test_wa_value_frozen():
    """test_wirelength.py:29."""
    val, _ = wl.wa_smooth([0.0, 10.0], 1.0)
    assert val == pytest.approx(9.999092042625951, rel=1e-12)


def test_wa_constant_set():
    """test_wirelength.py:35."""
    val, grad = wl.wa_smooth([3.0] * 5, 2.0)
    assert isinstance(grad, np.ndarray)
    assert val == pytest.approx(0.0, abs=1e-12)
    assert grad.sum() == pytest.approx(0.0, abs=1e-12)


def test_wa_gradient_finite_difference():
    """test_wirelength.py:41."""
    rng = np.random.default_rng(0)
    for _ in range(30):
        n = rng.integers(2, 8)
        v = rng.uniform(0, 50, n)
        gamma = rng.uniform(0.5, 5.0)
        _, grad = wl.wa_smooth(v, gamma)
        h = 1e-5
        for i in range(n):
            vp, vm = v.copy(), v.copy()
            vp[i] += h
            vm[i] -= h
            fd = (wl.wa_smooth(vp, gamma)[0] - wl.wa_smooth(vm, gamma)[0]) / (2 * h)
            assert grad[i] == pytest.approx(fd, rel=1e-5, abs=1e-9)


def test_wa_bounds_and_monotone_gamma():
    """test_wirelength.py:57."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        n = int(rng.integers(2, 9))
        v = rng.uniform(0, 100, n)
        span = v.max() - v.min()
        prev = -math.inf
        for k in range(6):
            gamma = 8.0 / (2 ** k)
            val, _ = wl.wa_smooth(v, gamma)
            assert -1e-9 <= val <= span + 1e-9
            assert span - val <= 2 * gamma * math.log(n) + 1e-9
            assert val >= prev - 1e-12
            prev = val


def brute_min_d2d_axis(coords, on_top):
    """test_wirelength.py:108-126: minimum over integer terminal positions."""
    coords = np.asarray(coords, dtype=float)
    top = coords[np.asarray(on_top, bool)]
    bot = coords[~np.asarray(on_top, bool)]
    if len(top) == 0 or len(bot) == 0:
        side = top if len(top) else bot
        return float(side.max() - side.min()) if len(side) else 0.0
    best = math.inf
    for t in range(int(coords.min()) - 1, int(coords.max()) + 2):
        best = min(best, max(top.max(), t) - min(top.min(), t) + max(bot.max(), t) - min(bot.min(), t))
    return best


def test_bistratal_fig4_configurations():
    """test_wirelength.py:129, :134."""
    assert wl.bistratal_axis([0, 1, 2, 3], [True, False, True, False]) == 4
    assert wl.bistratal_axis([0, 1, 2, 3], [True, True, False, False]) == 3
    assert wl.bistratal_axis([0, 7], [False, False]) == 7


def _nets(rng, count, lo, hi):
    sizes = [int(rng.integers(lo, hi)) for _ in range(count)]
    nets = [random_net(rng, n) for n in sizes]
    return sizes, nets


def test_bistratal_equals_brute_force():
    """test_wirelength.py:138 (500 random nets; here all 500 in one device
    launch, the same nets the reference draws one at a time)."""
    rng = np.random.default_rng(3)
    sizes, nets = [], []
    for _ in range(500):
        n = int(rng.integers(1, 9))
        sizes.append(n)
        nets.append(random_net(rng, n))
    topo = make_topo(sizes)
    coords = np.concatenate([c for c, _ in nets])
    on_top = np.concatenate([t for _, t in nets])
    got = wl.bistratal_spans(topo, coords, on_top)
    assert isinstance(got, np.ndarray)
    want = [brute_min_d2d_axis(c, t) for c, t in nets]
    assert np.array_equal(got, want)
    # and the one-net entry point on a sample
    for c, t in nets[:40]:
        assert wl.bistratal_axis(c, t) == brute_min_d2d_axis(c, t)


def test_bistratal_bounds():
    """test_wirelength.py:148."""
    rng = np.random.default_rng(4)
    for _ in range(300):
        n = int(rng.integers(2, 10))
        coords, on_top = random_net(rng, n)
        full = wl.partial_hpwl(coords)
        assert full <= wl.bistratal_axis(coords, on_top) <= 2 * full + 1e-12


def test_planar_objective_coincident_pins():
    """test_wirelength.py:161."""
    val, gx, gy = wl.planar_objective(make_topo([3]), np.zeros(3), np.zeros(3),
                                      np.array([True, False, True]), 1.0)
    assert val == pytest.approx(0.0, abs=1e-12)
    assert np.allclose(gx, 0) and np.allclose(gy, 0)


def test_planar_objective_single_die_reduces_to_wa():
    """test_wirelength.py:170."""
    x = np.array([0.0, 10.0])
    y = np.array([5.0, 5.0])
    val, gx, gy = wl.planar_objective(make_topo([2]), x, y, np.array([False, False]), 1.5)
    wx, gwx = wl.wa_smooth(x, 1.5)
    wy, _ = wl.wa_smooth(y, 1.5)
    assert val == pytest.approx(wx + wy, rel=1e-12)
    assert np.allclose(gx, gwx)


def test_planar_gradient_matches_finite_difference():
    """test_wirelength.py:182."""
    rng = np.random.default_rng(5)
    gamma = 2.0
    checked = 0
    while checked < 100:
        n = int(rng.integers(2, 8))
        x, on_top = random_net(rng, n, span=60)
        y, _ = random_net(rng, n, span=60)
        x = x + rng.uniform(0, 1, n)
        y = y + rng.uniform(0, 1, n)
        topo = make_topo([n])
        tx, bx, fx = wl.NetBoxes(topo, x, on_top).spans()
        ty, by, fy = wl.NetBoxes(topo, y, on_top).spans()
        if abs(tx + bx - fx) < 1e-2 or abs(ty + by - fy) < 1e-2:
            continue
        _, gx, _ = wl.planar_objective(topo, x, y, on_top, gamma)
        h = 1e-6 * max(60.0, np.abs(x).max())
        for i in range(n):
            xp, xm = x.copy(), x.copy()
            xp[i] += h
            xm[i] -= h
            fd = (wl.planar_objective(topo, xp, y, on_top, gamma)[0]
                  - wl.planar_objective(topo, xm, y, on_top, gamma)[0]) / (2 * h)
            assert gx[i] == pytest.approx(fd, rel=1e-4, abs=1e-7)
        checked += 1


def test_fd_z_naive_spec_example():
    """test_wirelength.py:213."""
    grad = wl.fd_z_gradient_naive(make_topo([4]), np.array([0.0, 1.0, 2.0, 3.0]), np.zeros(4),
                                  np.array([True, False, True, False]), 4.0)
    assert grad[2] == pytest.approx(1.0)


def test_fd_z_single_pin_net():
    """test_wirelength.py:223."""
    grad = wl.fd_z_gradient_naive(make_topo([1]), np.array([5.0]), np.array([1.0]),
                                  np.array([True]), 4.0)
    assert grad[0] == 0.0


def test_fd_z_interior_pin_zero():
    """test_wirelength.py:231."""
    grad = wl.fd_z_gradient_naive(make_topo([5]), np.array([0.0, 10.0, 5.0, 0.0, 10.0]),
                                  np.zeros(5), np.array([True, True, True, False, False]), 4.0)
    assert grad[2] == 0.0


def test_incremental_equals_naive_random():
    """test_wirelength.py:241 (1000 random nets, bit-equal)."""
    rng = np.random.default_rng(6)
    sizes = [int(rng.integers(1, 10)) for _ in range(1000)]
    topo = make_topo(sizes)
    x, y = np.zeros(topo.n_pin), np.zeros(topo.n_pin)
    on_top = np.zeros(topo.n_pin, dtype=bool)
    pos = 0
    for n in sizes:
        cx, ct = random_net(rng, n)
        cy, _ = random_net(rng, n)
        x[pos: pos + n], y[pos: pos + n], on_top[pos: pos + n] = cx, cy, ct
        pos += n
    naive = wl.fd_z_gradient_naive(topo, x, y, on_top, 4.0)
    inc = wl.fd_z_gradient_incremental(topo, x, y, on_top, 4.0)
    assert isinstance(inc, np.ndarray) and np.array_equal(naive, inc)


def test_incremental_handles_repeated_instance():
    """test_wirelength.py:264."""
    topo = wl.NetTopology(np.array([0, 3]), np.zeros(3, dtype=np.int64), np.array([0, 0, 1]), 2)
    args = (topo, np.array([0.0, 4.0, 2.0]), np.zeros(3), np.array([True, True, False]), 4.0)
    assert np.array_equal(wl.fd_z_gradient_naive(*args), wl.fd_z_gradient_incremental(*args))


def test_incremental_tie_at_boundary():
    """test_wirelength.py:278."""
    args = (make_topo([3]), np.array([0.0, 5.0, 5.0]), np.zeros(3), np.array([True] * 3), 4.0)
    assert np.array_equal(wl.fd_z_gradient_naive(*args), wl.fd_z_gradient_incremental(*args))


def test_normalize_cases():
    """test_wirelength.py:292, :300, :309."""
    out = wl.normalize_z_gradient(np.array([1.0, 2.0]), np.array([0.5, 0.5]), np.zeros(2),
                                  np.array([3.0, -1.0]), 0.5)
    assert np.allclose(out, 0.5 * np.array([3.0, -1.0]))
    gz = np.array([0.5, 0.5])
    out = wl.normalize_z_gradient(np.array([1.0, 0.0]), np.array([0.0, 1.0]), gz, np.zeros(2), 0.0)
    assert np.allclose(out, gz)
    out = wl.normalize_z_gradient(np.array([2.0, 0.0]), np.array([0.0, 2.0]), np.array([1.0, 1.0]),
                                  np.zeros(2), 0.0)
    assert np.allclose(out, [1.0, 1.0])


# ==== test_density.py ===============================================================


def test_dynamic_size_cases():
    """test_density.py:49, :57, :63, :71."""
    dz = 8.0
    w, h = dn.dynamic_size([4], [6], [2], [3], [True], [dz / 4], dz)
    assert isinstance(w, np.ndarray) and (w[0], h[0]) == (2, 3)
    w, h = dn.dynamic_size([4], [6], [2], [3], [True], [3 * dz / 4], dz)
    assert (w[0], h[0]) == (4, 6)
    w, _ = dn.dynamic_size([4], [4], [2], [2], [True], [dz / 2], dz)
    assert w[0] == pytest.approx(3.0)
    w, _ = dn.dynamic_size([4], [4], [2], [2], [False], [dz / 2 - 0.01], dz)
    assert w[0] == 2
    w, _ = dn.dynamic_size([4], [4], [2], [2], [False], [dz / 2 + 0.01], dz)
    assert w[0] == 4
    w, _ = dn.dynamic_size([4], [4], [2], [2], [True], [0.0], dz)
    assert w[0] == 2


def test_dynamic_size_macro_continuity():
    """test_density.py:77."""
    dz = 8.0
    zs = np.linspace(dz / 4, 3 * dz / 4, 501)
    w, _ = dn.dynamic_size([10], [10], [2], [2], [True], zs, dz)
    assert np.abs(np.diff(w)).max() <= (zs[1] - zs[0]) * 2 * 8 / dz + 1e-12


def test_direct_density_unit_cube_and_straddle():
    """test_density.py:89, :97."""
    grid = dn.DensityGrid(4, 4, 4, 4, 4)
    rho = dn.direct_density(grid, make_cloud([(1.5, 2.5, 3.5, 1, 1, 1)]))
    assert rho[1, 2, 3] == pytest.approx(1.0) and rho.sum() == pytest.approx(1.0)
    rho = dn.direct_density(grid, make_cloud([(2.0, 0.5, 0.5, 1, 1, 1)]))
    assert rho[1, 0, 0] == pytest.approx(0.5) and rho[2, 0, 0] == pytest.approx(0.5)


def test_direct_density_matches_brute_force():
    """test_density.py:105."""
    rng = np.random.default_rng(7)
    grid = dn.DensityGrid(8, 6, 4, 4, 4)
    boxes = []
    for _ in range(20):
        w, h = rng.uniform(0.3, 3), rng.uniform(0.3, 3)
        dep = rng.uniform(0.3, grid.dz / 2)
        boxes.append((rng.uniform(w / 2, 8 - w / 2), rng.uniform(h / 2, 6 - h / 2),
                      rng.uniform(dep / 2, grid.dz - dep / 2), w, h, dep))
    cloud = make_cloud(boxes, weights=rng.uniform(0.5, 2, 20))
    assert np.abs(dn.direct_density(grid, cloud) - brute_density(grid, cloud)).max() < 1e-9


def test_prefix_sum_cases():
    """test_density.py:147, :156, :162."""
    p = dn.prefix_sum_3d(np.ones((2, 2, 2)))
    for i in range(2):
        for j in range(2):
            for k in range(2):
                assert p[i, j, k] == (i + 1) * (j + 1) * (k + 1)
    a = np.zeros((3, 3, 3))
    a[0, 0, 0] = 1
    assert (dn.prefix_sum_3d(a) == 1).all()
    a = np.random.default_rng(8).normal(size=(3, 3, 3))
    p = dn.prefix_sum_3d(a)
    for i in range(3):
        for j in range(3):
            for k in range(3):
                assert p[i, j, k] == pytest.approx(a[: i + 1, : j + 1, : k + 1].sum(),
                                                   rel=1e-12, abs=1e-12)


def test_suffix_sum_is_prefix_adjoint():
    """test_density.py:173."""
    rng = np.random.default_rng(9)
    a = rng.normal(size=(4, 3, 5))
    b = rng.normal(size=(4, 3, 5))
    assert (dn.prefix_sum_3d(a) * b).sum() == pytest.approx((a * dn.suffix_sum_3d(b)).sum(),
                                                            rel=1e-12)


def test_macro_prefix_small_cases():
    """test_density.py:182, :191."""
    grid = dn.DensityGrid(2, 2, 2, 2, 2)
    rho = dn.macro_prefix_density(grid, make_cloud([(1.0, 0.5, 0.5, 2, 1, 1)], macro=[True]))
    assert rho[0, 0, 0] == pytest.approx(1.0) and rho[1, 0, 0] == pytest.approx(1.0)
    assert rho.sum() == pytest.approx(2.0)
    empty = make_cloud(np.zeros((0, 6)), macro=np.zeros(0, bool))
    assert (dn.macro_prefix_density(grid, empty) == 0).all()


def test_macro_prefix_theorem_oracle():
    """test_density.py:197 (50 random grids and macro sets)."""
    rng = np.random.default_rng(10)
    for _ in range(50):
        nx, ny, nz = rng.integers(2, 7, 3)
        dx, dy = rng.uniform(4, 20, 2)
        grid = dn.DensityGrid(dx, dy, int(nx), int(ny), int(nz))
        n_mac = int(rng.integers(1, 5))
        boxes = []
        for _ in range(n_mac):
            w, h = rng.uniform(0.5, dx), rng.uniform(0.5, dy)
            dep = grid.dz / 2
            boxes.append((rng.uniform(w / 2, dx - w / 2), rng.uniform(h / 2, dy - h / 2),
                          rng.uniform(dep / 2, grid.dz - dep / 2), w, h, dep))
        cloud = make_cloud(boxes, weights=rng.uniform(0.5, 2, n_mac), macro=[True] * n_mac)
        assert np.abs(dn.macro_prefix_density(grid, cloud) - brute_density(grid, cloud)).max() < 1e-9


def test_macro_grid_aligned_charge_conserved():
    """test_density.py:220."""
    grid = dn.DensityGrid(4, 4, 4, 4, 4)
    rho = dn.macro_prefix_density(grid, make_cloud([(2.0, 2.0, 2.0, 4, 4, 2)], weights=[0.7],
                                                   macro=[True]))
    assert np.allclose(rho[:, :, 1:3], 0.7)
    assert rho.sum() * grid.bin_vol == pytest.approx(0.7 * 4 * 4 * 2, rel=1e-12)


def test_accumulate_density_charge_conservation():
    """test_density.py:231."""
    rng = np.random.default_rng(11)
    grid = dn.DensityGrid(10, 8, 4, 4, 4)
    boxes = []
    for _ in range(30):
        w, h = rng.uniform(0.3, 4), rng.uniform(0.3, 4)
        dep = grid.dz / 2
        boxes.append((rng.uniform(w / 2, 10 - w / 2), rng.uniform(h / 2, 8 - h / 2),
                      rng.uniform(dep / 2, grid.dz - dep / 2), w, h, dep))
    macro = rng.random(30) < 0.3
    cloud = make_cloud(boxes, weights=rng.uniform(0.5, 2, 30), macro=macro)
    rho = dn.accumulate_density(grid, cloud)
    assert rho.sum() * grid.bin_vol == pytest.approx(float(cloud.charge.sum()), rel=1e-9)


def test_uniform_density_zero_potential():
    """test_density.py:254."""
    grid = dn.DensityGrid(8, 8, 8, 8, 8)
    phi, coef = dn.solve_potential(np.full(grid.shape, 0.7), grid)
    assert np.abs(phi).max() < 1e-12
    ex, ey, ez = dn.electric_field(coef, grid)
    assert np.abs(ex).max() < 1e-12 and np.abs(ez).max() < 1e-12


def _centers(grid):
    return np.meshgrid((np.arange(grid.nx) + 0.5) * grid.wb, (np.arange(grid.ny) + 0.5) * grid.hb,
                       (np.arange(grid.nz) + 0.5) * grid.db, indexing="ij")


def test_eigenfunction_recovery():
    """test_density.py:270."""
    rng = np.random.default_rng(12)
    grid = dn.DensityGrid(12.5, 9.0, 16, 16, 16)
    X, Y, Z = _centers(grid)
    wx, wy, wz = grid.omega
    for _ in range(10):
        j, k, l = (int(rng.integers(0, 16)) for _ in range(3))
        if (j, k, l) == (0, 0, 0):
            j = 1
        rho = np.cos(wx[j] * X) * np.cos(wy[k] * Y) * np.cos(wz[l] * Z)
        phi, _ = dn.solve_potential(rho, grid)
        lam = wx[j] ** 2 + wy[k] ** 2 + wz[l] ** 2
        assert np.abs(phi - rho / lam).max() < 1e-6 * np.abs(rho / lam).max()


def test_field_eigenfunction():
    """test_density.py:285."""
    grid = dn.DensityGrid(10.0, 10.0, 16, 16, 8)
    X, _, _ = _centers(grid)
    w1 = grid.omega[0][1]
    _, coef = dn.solve_potential(np.cos(w1 * X), grid)
    ex, ey, ez = dn.electric_field(coef, grid)
    assert np.abs(ex - np.sin(w1 * X) / w1).max() < 1e-9
    assert np.abs(ey).max() < 1e-9 and np.abs(ez).max() < 1e-9


def test_poisson_residual_spectral_operator():
    """test_density.py:297."""
    rng = np.random.default_rng(13)
    grid = dn.DensityGrid(8, 8, 8, 8, 8)
    rho = rng.uniform(0, 2, grid.shape)
    phi, _ = dn.solve_potential(rho, grid)
    wx, wy, wz = grid.omega
    lam = wx[:, None, None] ** 2 + wy[None, :, None] ** 2 + wz[None, None, :] ** 2
    lap = sfft.idctn(sfft.dctn(phi, type=2) * -lam, type=2)
    target = -(rho - rho.mean())
    assert np.linalg.norm(lap - target) / np.linalg.norm(target) < 1e-2


def test_field_matches_phi_derivative():
    """test_density.py:313."""
    rng = np.random.default_rng(14)
    grid = dn.DensityGrid(16.0, 12.0, 16, 16, 16)
    X, Y, Z = _centers(grid)
    wx, wy, wz = grid.omega
    rho = np.zeros(grid.shape)
    for _ in range(8):
        j, k, l = (int(rng.integers(0, 4)) for _ in range(3))
        rho += rng.normal() * np.cos(wx[j] * X) * np.cos(wy[k] * Y) * np.cos(wz[l] * Z)
    phi, coef = dn.solve_potential(rho, grid)
    fields = dn.electric_field(coef, grid)
    pad = np.pad(phi, 2, mode="symmetric")
    steps = (grid.wb, grid.hb, grid.db)
    for axis in range(3):
        def shift(o):
            s = [slice(2, -2)] * 3
            s[axis] = slice(2 + o, pad.shape[axis] - 2 + o)
            return pad[tuple(s)]

        e_fd = -(-shift(2) + 8 * shift(1) - 8 * shift(-1) + shift(-2)) / (12 * steps[axis])
        rel = np.linalg.norm(e_fd - fields[axis]) / max(np.linalg.norm(fields[axis]), 1e-30)
        assert rel < 0.02


def _solve(grid, cloud):
    rho = dn.accumulate_density(grid, cloud)
    phi, coef = dn.solve_potential(rho, grid)
    ex, ey, ez = dn.electric_field(coef, grid)
    return rho, phi, ex, ey, ez


def test_symmetric_pair_opposite_forces():
    """test_density.py:352."""
    grid = dn.DensityGrid(16, 16, 16, 16, 8)
    cloud = make_cloud([(8.0 - 1.3, 8, grid.dz / 2, 2, 2, grid.dz / 2),
                        (8.0 + 1.3, 8, grid.dz / 2, 2, 2, grid.dz / 2)])
    _, phi, ex, ey, ez = _solve(grid, cloud)
    _, grad = dn.density_energy_and_gradient(grid, cloud, phi, ex, ey, ez)
    assert isinstance(grad, np.ndarray)
    assert grad[0, 0] == pytest.approx(-grad[1, 0], rel=1e-9)
    assert grad[0, 0] > 0 and grad[1, 0] < 0


def test_macro_gradient_matches_direct_path():
    """test_density.py:367."""
    rng = np.random.default_rng(15)
    grid = dn.DensityGrid(16, 12, 8, 8, 8)
    for _ in range(10):
        w, h = rng.uniform(2, 8), rng.uniform(2, 6)
        box = (rng.uniform(w / 2, 16 - w / 2), rng.uniform(h / 2, 12 - h / 2),
               rng.uniform(grid.dz / 4, 3 * grid.dz / 4), w, h, grid.dz / 2)
        filler = (4.0, 3.0, grid.dz / 4, 1.5, 1.5, grid.dz / 2)
        as_macro = make_cloud([box, filler], macro=[True, False])
        as_cell = make_cloud([box, filler], macro=[False, False])
        _, phi, ex, ey, ez = _solve(grid, as_macro)
        _, g1 = dn.density_energy_and_gradient(grid, as_macro, phi, ex, ey, ez)
        _, g2 = dn.density_energy_and_gradient(grid, as_cell, phi, ex, ey, ez)
        assert np.abs(g1 - g2).max() < 1e-9


def test_force_balance_mirrored_state():
    """test_density.py:386."""
    rng = np.random.default_rng(16)
    grid = dn.DensityGrid(16, 16, 8, 8, 8)
    boxes = []
    for _ in range(12):
        w, h = rng.uniform(0.5, 3), rng.uniform(0.5, 3)
        x, y = rng.uniform(w / 2, 8 - w / 2), rng.uniform(h / 2, 16 - h / 2)
        z = rng.uniform(grid.dz / 4, 3 * grid.dz / 4)
        boxes.append((x, y, z, w, h, grid.dz / 2))
        boxes.append((16 - x, y, z, w, h, grid.dz / 2))
    cloud = make_cloud(boxes)
    _, phi, ex, ey, ez = _solve(grid, cloud)
    _, grad = dn.density_energy_and_gradient(grid, cloud, phi, ex, ey, ez)
    assert abs(grad[:, 0].sum()) <= 1e-6 * max(np.abs(grad[:, 0]).sum(), 1e-30)


def test_energy_gradient_matches_finite_difference():
    """test_density.py:408."""
    rng = np.random.default_rng(17)
    grid = dn.DensityGrid(16, 16, 16, 16, 16)
    boxes = [(int(rng.integers(4, 12)) + rng.uniform(0.3, 0.7),
              int(rng.integers(4, 12)) + rng.uniform(0.3, 0.7),
              grid.dz * 0.5 + rng.uniform(-2, 2), 2.5, 2.5, grid.dz / 2) for _ in range(6)]
    cloud = make_cloud(boxes)

    def energy_at(xs, ys):
        c = make_cloud(boxes)
        c.x[:] = xs
        c.y[:] = ys
        _, phi, ex, ey, ez = _solve(grid, c)
        return dn.density_energy_and_gradient(grid, c, phi, ex, ey, ez)[0]

    _, phi, ex, ey, ez = _solve(grid, cloud)
    _, grad = dn.density_energy_and_gradient(grid, cloud, phi, ex, ey, ez)
    h = 0.01
    for i in range(len(boxes)):
        for axis in (0, 1):
            xs, ys = cloud.x.copy(), cloud.y.copy()
            arr = xs if axis == 0 else ys
            arr[i] += h
            up = energy_at(xs, ys)
            arr[i] -= 2 * h
            fd = (up - energy_at(xs, ys)) / (2 * h)
            assert grad[i, axis] == pytest.approx(fd, rel=0.02, abs=1e-9)


def test_overflow_cases():
    """test_density.py:445."""
    grid = dn.DensityGrid(4, 4, 4, 4, 4)
    assert dn.overflow(np.full(grid.shape, 0.5), grid, 1.0, 10.0) == 0.0
    assert dn.overflow(np.full(grid.shape, 1.0), grid, 1.0, 10.0) == 0.0
    rho = np.zeros(grid.shape)
    rho[0, 0, 0] = 3.0
    mv = 3.0 * grid.bin_vol
    assert dn.overflow(rho, grid, 1.0, mv) == pytest.approx(2.0 * grid.bin_vol / mv)


# ==== test_gp.py ========================================================================


def test_precondition_examples():
    """test_gp.py:13."""
    out, div = gpm.precondition(np.ones((3, 3)), 1.0, charges=np.array([0.3, 0.3, 7.0]),
                                pin_degrees=np.array([5.0, 2.0, 3.0]),
                                macro_flags=np.array([True, False, False]))
    assert div[0] == pytest.approx(5.3) and div[1] == 1.0 and div[2] == pytest.approx(7.0)
    assert np.allclose(out[0], 1 / 5.3) and np.allclose(out[2], 1 / 7.0)


def test_precondition_all_divisors_at_least_one():
    """test_gp.py:29."""
    rng = np.random.default_rng(0)
    _, div = gpm.precondition(rng.normal(size=(50, 3)), 1e-6, rng.uniform(0, 5, 50),
                              rng.integers(0, 9, 50), rng.random(50) < 0.3)
    assert (div >= 1).all()


def test_nesterov_zero_gradient_no_move():
    """test_gp.py:108."""
    opt = gpm.NesterovOptimizer(np.array([1.0, 2.0]))
    assert np.array_equal(opt.advance(np.zeros(2)), [1.0, 2.0])


def test_nesterov_quadratic_convergence():
    """test_gp.py:114."""
    rng = np.random.default_rng(1)
    t = rng.uniform(-5, 5, 8)
    d = rng.uniform(0.5, 4.0, 8)
    opt = gpm.NesterovOptimizer(np.zeros(8))
    x = opt.u
    for it in range(200):
        x = opt.advance(d * (opt.v - t), step_scale=1.0)
        if np.abs(x - t).max() < 1e-8:
            break
    assert np.abs(x - t).max() < 1e-6 and it < 199


def test_nesterov_projection_clamps():
    """test_gp.py:130."""
    opt = gpm.NesterovOptimizer(np.array([2.0]), project=lambda p: np.maximum(p, 1.0))
    assert opt.advance(np.array([100.0]), step_scale=1.0)[0] == 1.0


def _mixed_design(seed=0, n=60):
    """test_gp.py:140 (place3d.synth.gen_design; synth_arrays reproduces its
    arrays bit for bit, tests/test_synth.py)."""
    return synth_arrays(SynthSpec(n_insts=n, n_macros=2, r_ma=0.25, seed=seed))


def _problem(design, cfg, rng):
    grid = gpm.choose_grid(design, cfg)
    state = gpm.init_state(design, grid, cfg, rng)
    state.fillers = gpm.make_fillers(design, grid, rng)
    prob = gpm.Gp3dProblem(design, grid, state.fillers, cfg, state.rot)
    pos = np.zeros((prob.n_obj, 3))
    pos[: prob.n_inst] = np.c_[state.x, state.y, state.z]
    pos[prob.n_inst:] = np.c_[state.fillers.x, state.fillers.y, state.fillers.z]
    return grid, prob, pos


def test_assemble_lambda_zero_pure_wirelength():
    """test_gp.py:158."""
    cfg = gpm.GpConfig(seed=0)
    grid, prob, pos = _problem(_mixed_design(), cfg, np.random.default_rng(0))
    bundle, *_ = prob.evaluate(pos, 0.0, grid.db)
    assert isinstance(bundle.total, np.ndarray)
    assert np.allclose(bundle.total, bundle.wl_grad)
    assert np.allclose(bundle.wl_grad[prob.n_inst:], 0.0)


def test_assemble_fillers_z_frozen():
    """test_gp.py:167."""
    cfg = gpm.GpConfig(seed=0)
    grid, prob, pos = _problem(_mixed_design(), cfg, np.random.default_rng(0))
    bundle, *_ = prob.evaluate(pos, 1.0, grid.db)
    assert np.allclose(bundle.dens_grad[prob.n_inst:, 2], 0.0)


def test_assemble_descent_direction_probe():
    """test_gp.py:174."""
    cfg = gpm.GpConfig(seed=0)
    rng = np.random.default_rng(3)
    grid, prob, _ = _problem(_mixed_design(), cfg, rng)
    lam, hits, trials = 1e-5, 0, 20
    for _ in range(trials):
        pos = np.zeros((prob.n_obj, 3))
        pos[:, 0] = rng.uniform(20, grid.dx - 20, prob.n_obj)
        pos[:, 1] = rng.uniform(20, grid.dy - 20, prob.n_obj)
        pos[:, 2] = rng.uniform(grid.dz / 4, 3 * grid.dz / 4, prob.n_obj)
        pos = prob.project(pos)
        bundle, *_ = prob.evaluate(pos, lam, grid.db)
        pre, _ = gpm.precondition(bundle.total, lam, prob.cloud(pos).charge, prob.degree_obj,
                                  prob.is_macro_obj)
        step = 1e-3 * grid.wb / max(np.abs(pre).max(), 1e-12)
        bundle2, *_ = prob.evaluate(prob.project(pos - step * pre), lam, grid.db)
        hits += bundle2.value < bundle.value
    assert hits >= 0.95 * trials


def test_run_gp3d_single_instance():
    """test_gp.py:202."""
    k = make_kind("c", 4, 4, [("p", 0, 0)])
    d = make_design([k], [k], [("a", "c", False)], [("n", [(0, "p")])], die=(64, 64), rows=(4, 4))
    cfg = gpm.GpConfig(seed=1, max_iters=50)
    rng = np.random.default_rng(1)
    grid = gpm.choose_grid(d, cfg)
    state = gpm.init_state(d, grid, cfg, rng)
    state, info = gpm.run_gp3d(d, state, cfg, grid=grid, rng=rng)
    assert info.final_overflow <= cfg.stop_overflow
    assert info.iterations <= 3
    assert 2 <= state.x[0] <= 62
    assert state.z[0] in (grid.dz / 4, 3 * grid.dz / 4)


def test_run_gp3d_rounds_z_and_preserves_crossings():
    """test_gp.py:217."""
    d = _mixed_design(seed=4, n=50)
    cfg = gpm.GpConfig(seed=2, max_iters=300)
    rng = np.random.default_rng(2)
    grid = gpm.choose_grid(d, cfg)
    state = gpm.init_state(d, grid, cfg, rng)
    state, _ = gpm.run_gp3d(d, state, cfg, grid=grid, rng=rng)
    assert set(np.unique(state.z)) <= {grid.dz / 4, 3 * grid.dz / 4}
    assert set(np.unique(partition_from_z(state.z, grid.dz))) <= {0, 1}


def test_run_gp2d_no_crossing_nets_decoupled():
    """test_gp.py:229."""
    from paper_2403_09070_b200.gp2d import run_gp2d_multi

    k = make_kind("c", 4, 4, [("p", 0, 0), ("q", 1, 0)])
    d = make_design([k], [k], [("a", "c", False), ("b", "c", False), ("c0", "c", False),
                               ("d", "c", False)],
                    [("n0", [(0, "p"), (1, "q")]), ("n1", [(2, "p"), (3, "q")])],
                    die=(64, 64), rows=(4, 4))
    cfg = gpm.GpConfig(seed=1, max_iters=120)
    state = PlacementState(x=np.array([20.0, 30.0, 25.0, 35.0]), y=np.full(4, 32.0),
                           z=np.array([6.0, 6.0, 2.0, 2.0]), rot=np.zeros(4, dtype=int), dz=8.0)
    state, info, hbts = run_gp2d_multi(d, state, cfg, rng=np.random.default_rng(1))
    assert hbts == {}
    assert info.final_overflow <= cfg.stop_overflow


def test_run_gp2d_hbt_converges_to_optimal_region():
    """test_gp.py:251."""
    from paper_2403_09070_b200.gp2d import run_gp2d_multi

    k = make_kind("c", 4, 4, [("p", 0, 0)])
    d = make_design([k], [k], [("a", "c", False), ("b", "c", False)],
                    [("n", [(0, "p"), (1, "p")])], die=(64, 64), rows=(4, 4), hbt=(2, 0, 10.0))
    state = PlacementState(x=np.array([16.0, 48.0]), y=np.array([32.0, 32.0]),
                           z=np.array([6.0, 2.0]), rot=np.zeros(2, dtype=int), dz=8.0)
    cfg = gpm.GpConfig(seed=1, max_iters=150)
    state, info, hbts = run_gp2d_multi(d, state, cfg, rng=np.random.default_rng(1))
    assert set(hbts) == {0}
    hx, hy = hbts[0]
    lo, hi = sorted([state.x[0], state.x[1]])
    assert lo - 2 <= hx <= hi + 2
    assert abs(hy - 32.0) <= 4.0


# ==== edge cases beyond the reference's own tests ========================================


def test_density_boxes_clipped_at_the_region_boundary():
    """Charges straddling or outside the region's faces (the reference clips
    each box to [0, dx] x [0, dy] x [0, dz], density.py:155-169): the device
    maps (direct and per-macro tile paths) equal the brute-force overlap
    integration, which clips the same way."""
    rng = np.random.default_rng(31)
    grid = dn.DensityGrid(10, 8, 5, 4, 2)
    boxes = []
    for _ in range(40):
        w, h = rng.uniform(0.5, 6), rng.uniform(0.5, 6)
        dep = rng.uniform(0.5, grid.dz)
        boxes.append((rng.uniform(-2, 12), rng.uniform(-2, 10), rng.uniform(-1, grid.dz + 1),
                      w, h, dep))
    weights = rng.uniform(0.5, 2, 40)
    want = brute_density(grid, make_cloud(boxes, weights=weights))
    got_cells = dn.direct_density(grid, make_cloud(boxes, weights=weights))
    got_macros = dn.macro_prefix_density(grid, make_cloud(boxes, weights=weights, macro=[True] * 40))
    assert np.abs(got_cells - want).max() < 1e-9
    assert np.abs(got_macros - want).max() < 1e-9


def test_wa_extreme_spread_is_finite():
    """A net spanning ~1e6 gammas: the shifted exponentials underflow to 0
    for the far pins (wirelength.py:64-66 shifts by the max / min), the value
    tends to the span and the gradient to +-1 at the extremes; nothing is
    non-finite."""
    v = np.array([0.0, 1.0, 5e5, 1e6])
    val, grad = wl.wa_smooth(v, 1.0)
    assert np.isfinite(val) and np.all(np.isfinite(grad))
    # wirelength.py:58-73 in numpy
    ep, em = np.exp(v - v.max()), np.exp(v.min() - v)
    vp, vm = (v * ep).sum() / ep.sum(), (v * em).sum() / em.sum()
    want = ep / ep.sum() * (1 + (v - vp)) - em / em.sum() * (1 - (v - vm))
    assert val == pytest.approx(vp - vm, rel=1e-12)
    assert np.allclose(grad, want, rtol=1e-9, atol=1e-12)
