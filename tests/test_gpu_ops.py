"""Per-operator parity of the CUDA path (through the C-ABI) against the
reference's own outputs (tests/golden/small_ops.npz, produced by place3d) and
the CPU oracle on seeded inputs.

Tolerances: the kernels compute in float64, so WL/density values and
gradients are compared at 1e-9 relative (north_star asks 1e-5 for fp32);
box extrema, the finite-difference depth gradient, spans and crossing counts
are compared bit-exactly; the fixed-point density map bit-exactly against
oracle.fixed.
"""

import os

import numpy as np
import pytest

from oracle import fixed as FX
from oracle import port as P

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def cpu(t):
    # numpy inputs give numpy results (the per-op drop-in convention)
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


@pytest.fixture(scope="module")
def small():
    from paper_2403_09070_b200.synth import SynthSpec, synth_arrays

    g = dict(np.load(os.path.join(GOLD, "small_ops.npz")))
    design = synth_arrays(SynthSpec(n_insts=2000, n_macros=6, r_ma=0.30, seed=3,
                                    nets_per_inst=1.2))
    return design, g


# ---------------------------------------------------------------------------
# K1 wirelength
# ---------------------------------------------------------------------------


def test_pin_coords_exact(small):
    from paper_2403_09070_b200 import wirelength as wl

    d, g = small
    n = d.n_insts
    pos = g["pos"]
    grid = P.Grid(d.die.width, d.die.height, 64, 64, 2)
    px, py, pz, top = wl.dynamic_pin_coords(d.arrays(), pos[:n, 0], pos[:n, 1], pos[:n, 2],
                                            np.zeros(n, np.int64), grid.dz)
    assert np.array_equal(cpu(px), g["px"]) and np.array_equal(cpu(py), g["py"])
    assert np.array_equal(cpu(pz), g["pz"]) and np.array_equal(cpu(top), g["top"])


def test_netboxes_exact(small):
    from paper_2403_09070_b200 import wirelength as wl

    d, g = small
    topo = wl.NetTopology.from_arrays(d.arrays())
    for ax in ("x", "y"):
        b = wl.NetBoxes(topo, g["p" + ax], g["top"])
        for f in ("cnt", "min1", "min2", "max1", "max2"):
            assert np.array_equal(cpu(getattr(b, f)), g[f"b{ax}_{f}"]), (ax, f)


def test_planar_objective(small):
    from paper_2403_09070_b200 import wirelength as wl

    d, g = small
    topo = wl.NetTopology.from_arrays(d.arrays())
    v, gx, gy = wl.planar_objective(topo, g["px"], g["py"], g["top"], float(g["gamma"]))
    assert abs(v - float(g["wl_value"])) <= 1e-12 * abs(float(g["wl_value"]))
    assert rel(gx, g["gx_pin"]) < 1e-12 and rel(gy, g["gy_pin"]) < 1e-12


def test_z_cut_penalty(small):
    from paper_2403_09070_b200 import wirelength as wl

    d, g = small
    topo = wl.NetTopology.from_arrays(d.arrays())
    v, gc = wl.z_cut_penalty(topo, g["pz"], float(g["gamma"]))
    assert abs(v - float(g["cut_value"])) <= 1e-12 * abs(float(g["cut_value"]))
    assert rel(gc, g["gcut_pin"]) < 1e-12


def test_fd_z_gradient_exact(small):
    from paper_2403_09070_b200 import wirelength as wl

    d, g = small
    a = d.arrays()
    topo = wl.NetTopology.from_arrays(a)
    grid = P.Grid(d.die.width, d.die.height, 64, 64, 2)
    gz = wl.fd_z_gradient_incremental(topo, g["px"], g["py"], g["top"], grid.dz,
                                      a.net_has_dup_inst)
    assert np.array_equal(cpu(gz), g["gz_bist"])


def _make_topo(sizes):
    from paper_2403_09070_b200 import wirelength as wl

    ptr = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=ptr[1:])
    n = int(ptr[-1])
    return wl.NetTopology(ptr, np.repeat(np.arange(len(sizes)), sizes), np.arange(n), n)


def _random_net(rng, n, span=100):
    base = rng.integers(0, span, n).astype(float)
    if n >= 2 and rng.random() < 0.4:
        base[rng.integers(0, n)] = base.max()
    top = rng.random(n) < rng.uniform(0.1, 0.9)
    return base, top


def test_incremental_equals_naive_random():
    """test_wirelength.py:241-261 on the device: 1,000 random integer nets."""
    from paper_2403_09070_b200 import wirelength as wl

    rng = np.random.default_rng(6)
    sizes = [int(rng.integers(1, 10)) for _ in range(1000)]
    topo = _make_topo(sizes)
    x = np.zeros(topo.n_pin)
    y = np.zeros(topo.n_pin)
    top = np.zeros(topo.n_pin, bool)
    p = 0
    for s in sizes:
        cx, ct = _random_net(rng, s)
        cy, _ = _random_net(rng, s)
        x[p:p + s], y[p:p + s], top[p:p + s] = cx, cy, ct
        p += s
    naive = wl.fd_z_gradient_naive(topo, x, y, top, 4.0)
    inc = wl.fd_z_gradient_incremental(topo, x, y, top, 4.0)
    ref = P.fd_depth_grad_naive(topo.net_ptr, topo.pin_inst, topo.n_obj, x, y, top, 4.0)
    assert np.array_equal(cpu(naive), cpu(inc))
    assert np.array_equal(cpu(inc), ref)


def test_repeated_instance_and_tie():
    """test_wirelength.py:264-286."""
    from paper_2403_09070_b200 import wirelength as wl

    topo = wl.NetTopology(np.array([0, 3]), np.zeros(3, np.int64), np.array([0, 0, 1]), 2)
    x, y, t = np.array([0.0, 4.0, 2.0]), np.zeros(3), np.array([True, True, False])
    assert np.array_equal(cpu(wl.fd_z_gradient_naive(topo, x, y, t, 4.0)),
                          cpu(wl.fd_z_gradient_incremental(topo, x, y, t, 4.0)))
    topo = _make_topo([3])
    x, t = np.array([0.0, 5.0, 5.0]), np.array([True, True, True])
    assert np.array_equal(cpu(wl.fd_z_gradient_naive(topo, x, y, t, 4.0)),
                          cpu(wl.fd_z_gradient_incremental(topo, x, y, t, 4.0)))
    # spec example (test_wirelength.py:213-220)
    topo = _make_topo([4])
    g = wl.fd_z_gradient_naive(topo, np.array([0.0, 1.0, 2.0, 3.0]), np.zeros(4),
                               np.array([True, False, True, False]), 4.0)
    assert cpu(g)[2] == pytest.approx(1.0)


def test_known_answers():
    from paper_2403_09070_b200 import wirelength as wl

    val, _ = wl.wa_smooth([0.0, 10.0], 1.0)
    assert val == pytest.approx(9.999092042625951, rel=1e-12)  # test_wirelength.py:29-32
    assert wl.bistratal_axis([0, 1, 2, 3], [True, False, True, False]) == 4  # :129-131
    assert wl.bistratal_axis([0, 1, 2, 3], [True, True, False, False]) == 3
    out = wl.normalize_z_gradient(np.array([2.0, 0.0]), np.array([0.0, 2.0]),
                                  np.array([1.0, 1.0]), np.zeros(2), 0.0)
    assert np.allclose(cpu(out), [1.0, 1.0])  # :309-314
    out = wl.normalize_z_gradient(np.array([1.0, 2.0]), np.array([0.5, 0.5]), np.zeros(2),
                                  np.array([3.0, -1.0]), 0.5)
    assert np.allclose(cpu(out), [1.5, -0.5])  # :292-299


def test_wa_gradient_vs_oracle_random():
    from paper_2403_09070_b200 import wirelength as wl

    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(1, 9))
        v = rng.uniform(0, 50, n)
        gamma = rng.uniform(0.5, 5.0)
        val, g = wl.wa_smooth(v, gamma)
        rv, rg = P.wa_one(v, gamma)
        assert val == pytest.approx(rv, rel=1e-12, abs=1e-12)
        assert np.allclose(cpu(g), rg, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------------------
# K2/K3/K4 density
# ---------------------------------------------------------------------------


def _small_cloud(small):
    d, g = small
    from paper_2403_09070_b200 import gp as G

    cfg = G.GpConfig(seed=1, nz=2, grid_nx=64, grid_ny=64, max_iters=60, stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg)
    st = G.init_state(d, grid, cfg, rng)
    fill = G.make_fillers(d, grid, rng)
    og = P.Grid(d.die.width, d.die.height, 64, 64, 2)
    ofill = P.Fill(fill.x, fill.y, fill.z, fill.die, fill.w, fill.h, fill.dep)
    oprob = P.Problem(d, og, ofill, P.Cfg(nz=2, grid_nx=64, max_iters=60, stop_overflow=0.0),
                      st.rot)
    return grid, og, oprob.cloud(g["pos"]), oprob, fill, st


def test_density_fixed_point_bit_exact(small):
    from paper_2403_09070_b200 import density as dn

    grid, og, cl, *_ = _small_cloud(small)
    got = dn.accumulate_density_fx(grid, dn.ChargeCloud(cl.x, cl.y, cl.z, cl.w, cl.h, cl.dep,
                                                        cl.weight, cl.is_macro))
    want = FX.fixed_rho(og, cl)
    assert np.array_equal(cpu(got), want)


def test_loop_scatter_bit_exact(small):
    """The fused loop's K2 (tile sort + shared-memory windows) == oracle.fixed,
    at the golden point and at a spread-out point (windows vs bbox fallback)."""
    from paper_2403_09070_b200 import gp as G

    d, g = small
    grid, og, cl, oprob, fill, st = _small_cloud(small)
    cfg = G.GpConfig(seed=1, nz=2, grid_nx=64, grid_ny=64, max_iters=60, stop_overflow=0.0)
    prob = G.Gp3dProblem(d, grid, fill, cfg, st.rot)
    rng = np.random.default_rng(7)
    spread = oprob.project(np.c_[rng.uniform(0, d.die.width, len(g["pos"])),
                                 rng.uniform(0, d.die.height, len(g["pos"])), g["pos"][:, 2]])
    for pos in (g["pos"], spread):
        got = prob.density_fx(pos)
        want = FX.fixed_rho(og, oprob.cloud(pos))
        assert np.array_equal(cpu(got), want)


def test_density_vs_reference(small):
    from paper_2403_09070_b200 import density as dn

    d, g = small
    grid, og, cl, *_ = _small_cloud(small)
    rho = dn.accumulate_density(grid, dn.ChargeCloud(cl.x, cl.y, cl.z, cl.w, cl.h, cl.dep,
                                                     cl.weight, cl.is_macro))
    assert np.abs(cpu(rho) - g["rho"]).max() < 1e-9  # brute_density tolerance (test_density.py:120)


def test_spectral_vs_reference(small):
    from paper_2403_09070_b200 import density as dn

    d, g = small
    grid = dn.DensityGrid(d.die.width, d.die.height, 64, 64, 2)
    phi, coef = dn.solve_potential(g["rho"], grid)
    assert rel(coef, g["coef"]) < 1e-12
    assert rel(phi, g["phi"]) < 1e-10
    ex, ey, ez = dn.electric_field(g["coef"], grid)
    for a, k in ((ex, "ex"), (ey, "ey"), (ez, "ez")):
        assert rel(a, g[k]) < 1e-10, k


@pytest.mark.parametrize("shape", [(8, 8, 8), (16, 12, 4), (12, 10, 6), (5, 7, 3), (128, 64, 2),
                                   (512, 512, 2), (256, 1024, 2), (32, 16, 16), (1024, 256, 2),
                                   (64, 32, 1), (64, 32, 3), (8, 1024, 2), (16, 8, 5), (1024, 1024, 2)])
def test_spectral_vs_scipy_shapes(shape):
    """FFT path (powers of two) and direct path (others) against scipy.fft."""
    from paper_2403_09070_b200 import density as dn

    nx, ny, nz = shape
    rng = np.random.default_rng(nx * 100 + ny)
    grid = dn.DensityGrid(17.0, 13.0, nx, ny, nz)
    og = P.Grid(17.0, 13.0, nx, ny, nz)
    rho = rng.uniform(0, 2, (nx, ny, nz))
    phi, coef = dn.solve_potential(rho, grid)
    rphi, rcoef = P.potential(rho, og)
    assert rel(coef, rcoef) < 1e-12 and rel(phi, rphi) < 1e-10
    e = dn.electric_field(rcoef, grid)
    re = P.efield(rcoef, og)
    for a, b in zip(e, re):
        assert rel(a, b) < 1e-10


def test_eigenfunction_and_uniform():
    """test_density.py:254-294 restated on the device."""
    from paper_2403_09070_b200 import density as dn

    grid = dn.DensityGrid(8, 8, 8, 8, 8)
    phi, coef = dn.solve_potential(np.full(grid.shape, 0.7), grid)
    assert float(np.abs(cpu(phi)).max()) < 1e-12
    grid = dn.DensityGrid(10.0, 10.0, 16, 16, 8)
    xs = (np.arange(16) + 0.5) * grid.wb
    X = np.broadcast_to(xs[:, None, None], grid.shape)
    w1 = grid.omega[0][1]
    phi, coef = dn.solve_potential(np.cos(w1 * X), grid)
    ex, ey, ez = dn.electric_field(coef, grid)
    assert np.abs(cpu(ex) - np.sin(w1 * X) / w1).max() < 1e-9
    assert float(np.abs(cpu(ey)).max()) < 1e-9 and float(np.abs(cpu(ez)).max()) < 1e-9


def test_energy_force_vs_reference(small):
    from paper_2403_09070_b200 import density as dn

    d, g = small
    grid, og, cl, oprob, fill, st = _small_cloud(small)
    c = dn.ChargeCloud(cl.x, cl.y, cl.z, cl.w, cl.h, cl.dep, cl.weight, cl.is_macro)
    e = dn.density_energy(grid, c, g["phi"])
    assert e == pytest.approx(float(g["energy"]), rel=1e-10)
    f = dn.density_force(grid, c, g["ex"], g["ey"], g["ez"], freeze_z=oprob.freeze_z)
    assert rel(f, g["force"]) < 1e-10


def test_overflow_fixed_point(small):
    from paper_2403_09070_b200 import density as dn

    d, g = small
    grid, og, cl, oprob, *_ = _small_cloud(small)
    acc = FX.fixed_rho(og, cl)
    import torch

    got = dn.overflow_fx(torch.from_numpy(acc).cuda(), grid, 1.0, oprob.movable_volume)
    assert got == pytest.approx(float(g["ovfl"]), rel=1e-12)


# ---------------------------------------------------------------------------
# GP problem: evaluate / project / precondition
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
def test_evaluate_vs_reference(small, precision, tol):
    """Gp3dProblem.evaluate: fp64 WA at 1e-12, fp32 WA at the north_star's 1e-5."""
    from paper_2403_09070_b200 import gp as G

    d, g = small
    grid, og, cl, oprob, fill, st = _small_cloud(small)
    cfg = G.GpConfig(seed=1, nz=2, grid_nx=64, grid_ny=64, max_iters=60, stop_overflow=0.0)
    prob = G.Gp3dProblem(d, grid, fill, cfg, st.rot, precision=precision)
    assert prob.movable_volume == float(g["movable_volume"]) and prob.alpha == float(g["alpha"])
    b, ov, ex, nc = prob.evaluate(g["pos"], 1e-3, float(g["gamma"]))
    assert nc == int(g["ncross"]) and ex == float(g["exact"])  # exact in both modes
    assert ov == pytest.approx(float(g["ovfl"]), rel=1e-12)
    assert b.value == pytest.approx(float(g["value"]), rel=tol)
    w, wr = cpu(b.wl_grad), g["wl_grad"]
    assert rel(w[:, :2], wr[:, :2]) < tol
    # the FD depth term inside gz is exact; the Eq. 17 scale carries the planar L1 norms
    assert rel(w[:, 2], wr[:, 2]) < tol
    assert rel(b.dens_grad, g["dens_grad"]) < 1e-9
    assert rel(b.total, g["total"]) < max(tol, 1e-9)
    pre, div = G.precondition(b.total, 1e-3, prob.cloud(g["pos"]).charge, prob.degree_obj,
                              prob.is_macro_obj)
    assert rel(pre, g["pre"]) < 1e-9 and rel(div, g["div"]) < 1e-14
    assert np.array_equal(cpu(prob.project(g["pos"])), oprob.project(g["pos"]))


def test_precondition_examples():
    """test_gp.py:13-26."""
    from paper_2403_09070_b200 import gp as G

    out, div = G.precondition(np.ones((3, 3)), 1.0, np.array([0.3, 0.3, 7.0]),
                              np.array([5.0, 2.0, 3.0]), np.array([True, False, False]))
    d = cpu(div)
    assert d[0] == pytest.approx(5.3) and d[1] == 1.0 and d[2] == pytest.approx(7.0)
    assert np.allclose(cpu(out)[0], 1 / 5.3) and np.allclose(cpu(out)[2], 1 / 7.0)


# ---------------------------------------------------------------------------
# exact energy gradient (density_energy_and_gradient)
# ---------------------------------------------------------------------------


def _cloud_of(boxes, macro=None, weight=None):
    from paper_2403_09070_b200 import density as dn

    b = np.asarray(boxes, dtype=np.float64)
    n = len(b)
    return dn.ChargeCloud(b[:, 0].copy(), b[:, 1].copy(), b[:, 2].copy(), b[:, 3].copy(),
                          b[:, 4].copy(), b[:, 5].copy(),
                          np.ones(n) if weight is None else np.asarray(weight, float),
                          np.zeros(n, bool) if macro is None else np.asarray(macro, bool))


def _device_solve(grid, cloud):
    from paper_2403_09070_b200 import density as dn

    rho = dn.accumulate_density(grid, cloud)
    phi, coef = dn.solve_potential(rho, grid)
    return phi


def test_energy_gradient_vs_reference_golden():
    """Against the reference's own density_energy_and_gradient output
    (tests/golden/energy_grad.npz): cells, macros, clipped boxes, frozen z."""
    from paper_2403_09070_b200 import density as dn

    g = dict(np.load(os.path.join(GOLD, "energy_grad.npz")))
    grid = dn.DensityGrid(16.0, 12.0, 16, 12, 8)
    cl = dn.ChargeCloud(*(g["a_" + k] for k in ("x", "y", "z", "w", "h", "dep", "weight",
                                                "is_macro")))
    e, grad = dn.density_energy_and_gradient(grid, cl, g["a_phi"], freeze_z=g["a_freeze"])
    assert e == pytest.approx(float(g["a_energy"]), rel=1e-12)
    assert rel(grad, g["a_grad"]) < 1e-13
    assert np.all(cpu(grad)[g["a_freeze"], 2] == 0.0)


def test_energy_gradient_symmetric_pair_and_macro_path():
    """test_density.py:352-387 restated on the device: a mirrored pair feels
    opposite forces; a macro's stamp-form gradient equals the cell face form."""
    from paper_2403_09070_b200 import density as dn

    grid = dn.DensityGrid(16, 16, 16, 16, 8)
    c, a = 8.0, 1.3
    cloud = _cloud_of([(c - a, 8, grid.dz / 2, 2, 2, grid.dz / 2),
                       (c + a, 8, grid.dz / 2, 2, 2, grid.dz / 2)])
    _, grad = dn.density_energy_and_gradient(grid, cloud, _device_solve(grid, cloud))
    g = cpu(grad)
    assert g[0, 0] == pytest.approx(-g[1, 0], rel=1e-9) and g[0, 0] > 0 > g[1, 0]
    rng = np.random.default_rng(15)
    grid = dn.DensityGrid(16, 12, 8, 8, 8)
    for _ in range(10):
        w, h = rng.uniform(2, 8), rng.uniform(2, 6)
        box = (rng.uniform(w / 2, 16 - w / 2), rng.uniform(h / 2, 12 - h / 2),
               rng.uniform(grid.dz / 4, 3 * grid.dz / 4), w, h, grid.dz / 2)
        filler = (4.0, 3.0, grid.dz / 4, 1.5, 1.5, grid.dz / 2)
        as_macro = _cloud_of([box, filler], macro=[True, False])
        as_cell = _cloud_of([box, filler], macro=[False, False])
        phi = _device_solve(grid, as_macro)
        _, g1 = dn.density_energy_and_gradient(grid, as_macro, phi)
        _, g2 = dn.density_energy_and_gradient(grid, as_cell, phi)
        assert float(np.abs(cpu(g1) - cpu(g2)).max()) < 1e-9


def test_energy_gradient_matches_finite_difference():
    """test_density.py:407-440 restated: central differences of U (each probe a
    full device density + spectral solve) match the exact gradient."""
    from paper_2403_09070_b200 import density as dn

    rng = np.random.default_rng(17)
    grid = dn.DensityGrid(16, 16, 16, 16, 16)
    boxes = [(int(rng.integers(4, 12)) + rng.uniform(0.3, 0.7),
              int(rng.integers(4, 12)) + rng.uniform(0.3, 0.7),
              grid.dz * 0.5 + rng.uniform(-2, 2), 2.5, 2.5, grid.dz / 2) for _ in range(6)]
    cloud = _cloud_of(boxes)
    _, grad = dn.density_energy_and_gradient(grid, cloud, _device_solve(grid, cloud))
    grad = cpu(grad)

    def energy_at(i, axis, dx):
        b = [list(t) for t in boxes]
        b[i][axis] += dx
        c = _cloud_of(b)
        return dn.density_energy_and_gradient(grid, c, _device_solve(grid, c))[0]

    h = 0.01
    for i in range(len(boxes)):
        for axis in (0, 1):
            fd = (energy_at(i, axis, h) - energy_at(i, axis, -h)) / (2 * h)
            assert grad[i, axis] == pytest.approx(fd, rel=0.02, abs=1e-9)  # test_density.py:442


def _with_odd_nets(design):
    """The small design plus nets the synthetic generator never makes: degree
    1, degree 9 and 12, and nets where one instance owns several pins (the
    O(|P|^2) exact FD path, wirelength.py:280-292) — the fused loop's generic
    kernel."""
    from paper_2403_09070_b200.model import ArrayDesign, NetlistArrays

    a = design.arrays()
    rng = np.random.default_rng(21)
    I = a.n_inst
    extra = [rng.choice(I, 12, replace=False), rng.choice(I, 9, replace=False), [5],
             [7, 7, 11], [3, 9, 3, 14, 9], np.r_[rng.choice(I, 6, replace=False), 17, 17]]
    ptr = list(a.net_ptr)
    inst = list(a.pin_inst)
    ox = [list(a.ox_top), list(a.oy_top), list(a.ox_bot), list(a.oy_bot)]
    for net in extra:
        for i in net:
            inst.append(int(i))
            for k in range(4):
                ox[k].append(float(rng.integers(-6, 7)))
        ptr.append(len(inst))
    arr = NetlistArrays(is_macro=a.is_macro, w_top=a.w_top, h_top=a.h_top, w_bot=a.w_bot,
                        h_bot=a.h_bot, net_ptr=np.array(ptr), pin_inst=np.array(inst),
                        ox_top=np.array(ox[0]), oy_top=np.array(ox[1]), ox_bot=np.array(ox[2]),
                        oy_bot=np.array(ox[3]))
    return ArrayDesign(design.die, design.hbt, arr)


def test_generic_and_duplicate_owner_nets_in_the_loop(small):
    """evaluate + 25 loop iterations with degree-1/9/12 and duplicate-owner
    nets (fused loop: generic kernel) against the oracle."""
    from paper_2403_09070_b200 import gp as G

    d0, g = small
    d = _with_odd_nets(d0)
    assert d.arrays().net_has_dup_inst.sum() >= 3
    cfg = G.GpConfig(seed=1, nz=2, grid_nx=64, grid_ny=64, max_iters=25, stop_overflow=0.0)
    ocfg = P.Cfg(seed=1, nz=2, grid_nx=64, grid_ny=64, max_iters=25, stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg)
    st = G.init_state(d, grid, cfg, rng)
    fill = G.make_fillers(d, grid, rng)
    og = P.grid_for(d, ocfg)
    ofill = P.Fill(fill.x, fill.y, fill.z, fill.die, fill.w, fill.h, fill.dep)
    prob = G.Gp3dProblem(d, grid, fill, cfg, st.rot)
    oprob = P.Problem(d, og, ofill, ocfg, st.rot)
    n = d.n_insts
    pos = np.zeros((prob.n_obj, 3))
    pos[:n] = np.c_[st.x, st.y, st.z]
    pos[n:] = np.c_[fill.x, fill.y, fill.z]
    pos = oprob.project(pos)
    b, ov, ex, nc = prob.evaluate(pos, 1e-3, 2 * grid.db)
    e, ov2, ex2, nc2 = oprob.evaluate(pos, 1e-3, 2 * og.db)
    assert nc == nc2 and ex == pytest.approx(ex2, rel=1e-12) and ov == pytest.approx(ov2, rel=1e-12)
    assert rel(b.wl_grad, e.wl_grad) < 1e-12
    rows, orows = [], []
    st2 = G.PlacementState(x=st.x.copy(), y=st.y.copy(), z=st.z.copy(), rot=st.rot, dz=grid.dz,
                           fillers=fill)
    G.run_gp3d(d, st2, cfg, grid=grid, iteration_log=rows, rng=rng)
    P.run_loop(d, pos[:n, 0], pos[:n, 1], pos[:n, 2], st.rot, ofill, ocfg, og, log=orows)
    assert len(rows) == len(orows) == 25
    for r, o in zip(rows, orows):
        assert r[2] == o[2] and abs(r[1] - o[1]) <= 1e-9 * abs(o[1]) and abs(r[3] - o[3]) <= 1e-9
