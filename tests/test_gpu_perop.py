"""The small per-op pieces of the reference's operator API on the device
(p3d_ops.cu, p3d_post.cu), each against the oracle restatement (itself pinned
to the reference, tests/test_oracle.py), and the numpy-in / numpy-out
convention of the drop-in ops (a reference caller passing numpy arrays gets
numpy arrays back)."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import port as P

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _small():
    z = np.load(os.path.join(GOLD, "small_ops.npz"))
    from paper_2403_09070_b200.synth import SynthSpec, synth_arrays

    spec = json.load(open(os.path.join(GOLD, "small_log.json")))["spec"]
    return synth_arrays(SynthSpec(**spec)), z


def test_dynamic_size_matches_oracle():
    from paper_2403_09070_b200 import density as dn

    rs = np.random.default_rng(1)
    n, dz = 5000, 80.0
    wt, ht = rs.uniform(5, 900, n), rs.uniform(5, 900, n)
    wb, hb = rs.uniform(5, 900, n), rs.uniform(5, 900, n)
    mac = rs.random(n) < 0.2
    z = rs.uniform(-10, 90, n)
    z[:10] = dz / 2  # the midplane itself belongs to the bottom die
    w, h = dn.dynamic_size(wt, ht, wb, hb, mac, z, dz)
    assert isinstance(w, np.ndarray)
    rw, rh = P.size_at_depth(wt, ht, wb, hb, mac, z, dz)
    assert np.array_equal(w, rw) and np.array_equal(h, rh)


@pytest.mark.parametrize("shape", [(16, 8, 2), (33, 7, 3), (64, 64, 1)])
def test_prefix_suffix_sum_3d(shape):
    from paper_2403_09070_b200 import density as dn

    rs = np.random.default_rng(2)
    a = rs.integers(-1000, 1000, shape).astype(np.float64)  # integers: every order exact
    got = dn.prefix_sum_3d(a)
    assert np.array_equal(got, np.cumsum(np.cumsum(np.cumsum(a, 0), 1), 2))
    assert np.array_equal(dn.suffix_sum_3d(a), P.rev_cumsum3(a))
    f = rs.standard_normal(shape)
    assert np.allclose(dn.prefix_sum_3d(f), np.cumsum(np.cumsum(np.cumsum(f, 0), 1), 2),
                       rtol=1e-12, atol=1e-12)


def test_overflow_and_macro_overflow():
    from paper_2403_09070_b200 import density as dn

    d, z = _small()
    grid = dn.DensityGrid(d.die.width, d.die.height, 64, 64, 2)
    rho = z["rho"]
    got = dn.overflow(rho, grid, 1.0, float(z["movable_volume"]))
    want = P.overflow_of(rho, P.Grid(d.die.width, d.die.height, 64, 64, 2), 1.0,
                         float(z["movable_volume"]))
    assert got == pytest.approx(want, rel=1e-12)
    # macro-only map of the small design's charge cloud (density.py:620-627)
    rs = np.random.default_rng(5)
    n = 300
    mac = rs.random(n) < 0.1
    cl = dn.ChargeCloud(x=rs.uniform(100, d.die.width - 100, n),
                        y=rs.uniform(100, d.die.height - 100, n), z=np.full(n, grid.dz / 2),
                        w=np.where(mac, 180.0, 12.0), h=np.where(mac, 150.0, 40.0),
                        dep=np.full(n, grid.dz / 2), weight=np.ones(n), is_macro=mac)
    og = P.Grid(d.die.width, d.die.height, 64, 64, 2)
    big = P.Cloud(cl.x[mac], cl.y[mac], cl.z[mac], cl.w[mac], cl.h[mac], cl.dep[mac],
                  cl.weight[mac], cl.is_macro[mac])
    want = P.overflow_of(P.macro_rho(og, big), og, 1.0, float(big.volume.sum()))
    assert dn.macro_overflow(grid, cl, 1.0) == pytest.approx(want, rel=1e-9)


def test_netboxes_spans_and_numpy_io():
    from paper_2403_09070_b200 import wirelength as wl

    d, z = _small()
    arr = d.arrays()
    topo = wl.NetTopology.from_arrays(arr)
    bx = wl.NetBoxes(topo, z["px"], z["top"])
    assert isinstance(bx.min1, np.ndarray)
    ob = P.Boxes(arr.pin_net, arr.n_net, z["px"], z["top"])
    for g_, r_ in zip(bx.spans(), ob.spans()):
        assert isinstance(g_, np.ndarray) and np.array_equal(g_, r_)
    # numpy in -> numpy out; tensors in -> tensors out
    v, gx, gy = wl.planar_objective(topo, z["px"], z["py"], z["top"], float(z["gamma"]))
    assert isinstance(gx, np.ndarray) and isinstance(gy, np.ndarray)
    assert np.abs(gx - z["gx_pin"]).max() <= 1e-12 * np.abs(z["gx_pin"]).max()
    vt, gxt, _ = wl.planar_objective(topo, torch.from_numpy(z["px"]).cuda(),
                                     torch.from_numpy(z["py"]).cuda(), z["top"], float(z["gamma"]))
    assert isinstance(gxt, torch.Tensor) and gxt.is_cuda


def test_nesterov_optimizer_matches_oracle():
    from paper_2403_09070_b200.gp import NesterovOptimizer

    rs = np.random.default_rng(3)
    n = 4000
    A = rs.uniform(0.5, 2.0, (n, 3))
    b = rs.standard_normal((n, 3))
    x0 = rs.standard_normal((n, 3))
    lo, hi = -3.0, 3.0
    proj_np = lambda p: np.clip(p, lo, hi)  # noqa: E731
    proj_t = lambda p: torch.clamp(p, lo, hi)  # noqa: E731
    ref = P.Nesterov(x0, project=proj_np)
    opt = NesterovOptimizer(torch.from_numpy(x0).cuda(), project=proj_t)  # tensors in, tensors out
    prev_r = prev_t = None
    for k in range(12):
        gr = A * ref.v - b  # gradient of sum(A x^2 / 2 - b x) at the lookahead point
        gt = torch.from_numpy(A).cuda() * opt.v - torch.from_numpy(b).cuda()
        ref.advance(gr, step_scale=0.5, g_prev_reval=prev_r)
        opt.advance(gt, step_scale=0.5, g_prev_reval=prev_t)
        prev_r, prev_t = gr, gt
        assert opt.step == pytest.approx(ref.step, rel=1e-12), k
        assert np.abs(opt.u.cpu().numpy() - ref.u).max() <= 1e-12 * np.abs(ref.u).max(), k


@pytest.mark.parametrize("rotated", [False, True])
def test_gp_wirelength_objective_vs_oracle(rotated):
    """wirelength.gp_wirelength_objective (wirelength.py:345-358) on the
    device against the oracle's pieces (pins_at, planar_wl, zcut and
    np.bincount, each pinned to the reference): value to 1e-12, the
    per-instance sums to 1e-12 of their scale."""
    from paper_2403_09070_b200 import wirelength as wl
    from paper_2403_09070_b200.synth import CONFIGS, synth_arrays

    d = synth_arrays(CONFIGS[1]["spec"])
    a = d.arrays()
    rs = np.random.default_rng(9)
    dz, gamma, alpha = 47.52, 17.3, 0.37
    x = rs.uniform(0, d.die.width, a.n_inst)
    y = rs.uniform(0, d.die.height, a.n_inst)
    z = rs.uniform(dz / 4, 3 * dz / 4, a.n_inst)
    rot = rs.integers(0, 4, a.n_inst) if rotated else np.zeros(a.n_inst, dtype=np.int64)
    val, gx, gy = wl.gp_wirelength_objective(a, x, y, z, rot, dz, gamma, alpha)
    assert isinstance(gx, np.ndarray) and gx.shape == (a.n_inst,)
    px, py, pz, top = P.pins_at(a, x, y, z, rot, dz)
    w_bi, gxp, gyp = P.planar_wl(a.pin_net, a.n_net, px, py, top, gamma)
    w_cut, _ = P.zcut(a.pin_net, a.n_net, pz, gamma)
    want_gx = np.bincount(a.pin_inst, weights=gxp, minlength=a.n_inst)
    want_gy = np.bincount(a.pin_inst, weights=gyp, minlength=a.n_inst)
    assert val == pytest.approx(w_bi + alpha * w_cut, rel=1e-12)
    assert np.abs(gx - want_gx).max() <= 1e-12 * np.abs(want_gx).max()
    assert np.abs(gy - want_gy).max() <= 1e-12 * np.abs(want_gy).max()


def test_gp2d_names_in_gp_module():
    """The reference keeps Gp2dProblem and run_gp2d_multi in gp.py
    (gp.py:463-690); so does the drop-in's gp module (gp2d.py behind it)."""
    from paper_2403_09070_b200 import gp, gp2d

    assert gp.run_gp2d_multi is gp2d.run_gp2d_multi
    assert gp.Gp2dProblem is gp2d.Gp2dProblem
    from paper_2403_09070_b200.gp import run_gp2d_multi  # noqa: F401


def test_precondition_two_column_gradients():
    """gp.precondition on [n, 2] gradients (the GP2D step's shape): the
    reference's gradients / div[..., None] (gp.py:142-147) to the last ulp."""
    from paper_2403_09070_b200 import gp as G

    rs = np.random.default_rng(12)
    n = 5000
    g = rs.standard_normal((n, 2)) * 10.0
    q = rs.uniform(0, 4, n)
    deg = rs.integers(0, 30, n).astype(float)
    mac = rs.random(n) < 0.1
    lam = 0.37
    out, div = G.precondition(g, lam, q, deg, mac)
    want_div = np.maximum(lam * q + np.where(mac, deg, 0.0), 1.0)
    assert isinstance(out, np.ndarray) and out.shape == (n, 2)
    assert np.array_equal(div, want_div)
    assert np.abs(out - g / want_div[:, None]).max() <= 1e-15 * np.abs(g / want_div[:, None]).max()


def test_overflow_degenerate_volumes():
    """density.overflow with no movable volume and macro_overflow without
    macros both return 0.0, as the reference does (density.py:612-627)."""
    from paper_2403_09070_b200 import density as dn

    grid = dn.DensityGrid(8, 8, 4, 4, 2)
    rho = np.full(grid.shape, 3.0)
    assert dn.overflow(rho, grid, 1.0, 0.0) == 0.0
    assert dn.overflow(rho, grid, 1.0, -1.0) == 0.0
    cloud = dn.ChargeCloud(x=np.array([2.0]), y=np.array([2.0]), z=np.array([1.0]),
                           w=np.array([1.0]), h=np.array([1.0]), dep=np.array([1.0]),
                           weight=np.array([1.0]), is_macro=np.array([False]))
    assert dn.macro_overflow(grid, cloud, 1.0) == 0.0
