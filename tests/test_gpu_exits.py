"""The early exits of run_gp3d and the rotated second pass, against runs of
the reference itself (tests/golden/exits.json, tests/golden/make_golden.py
--exits).

  * non-finite objective -> best state (gp.py:388-393), provoked with
    mu_min = mu_max = 1e200 (lambda overflows by iteration 2);
  * divergence window (gp.py:409-422), with divergence_window = 1;
  * step underflow (gp.py:436-441), with NesterovOptimizer's min_step = 1.5
    (the design's BB step first drops below it at iteration 28);
  * a second run_gp3d pass with every macro quarter-turned (rot = 1, 2, 3),
    as flow.py:121-122 runs it after the rotation MILP.

Each case checks the log rows, GpInfo and the returned state (sum / min /
max of x, y, z and the filler coordinates) against the reference.
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "exits.json")))


def _design():
    from paper_2403_09070_b200.synth import SynthSpec, synth_arrays

    return synth_arrays(SynthSpec(**GOLD["spec"]))


def _check_rows(rows, ref, tol=1e-9):
    got = np.array(rows, dtype=float)
    ref = np.array(ref, dtype=float)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.array_equal(got[:, 0], ref[:, 0])
    assert np.array_equal(got[:, 2], ref[:, 2])
    assert np.all(np.abs(got[:, 1] - ref[:, 1]) <= tol * ref[:, 1])
    assert np.all(np.abs(got[:, 3] - ref[:, 3]) <= tol * np.maximum(ref[:, 3], 1e-3))


def _check_info(info, ref, tol=1e-9):
    it, ovfl, div, wl, hbt = ref
    assert info.iterations == it
    assert bool(info.diverged) == div
    assert info.hbt_count == hbt
    assert info.final_overflow == pytest.approx(ovfl, rel=tol)
    assert info.wirelength == pytest.approx(wl, rel=tol)


def _check_state(st, ref, tol=1e-9):
    got = {"x": [st.x.sum(), st.x.min(), st.x.max()], "y": [st.y.sum(), st.y.min(), st.y.max()],
           "z": [st.z.sum()], "fx": [st.fillers.x.sum()], "fy": [st.fillers.y.sum()]}
    for k, v in ref.items():
        assert np.allclose(got[k], v, rtol=tol, atol=0), (k, got[k], v)


@pytest.mark.parametrize("case", sorted(GOLD["cases"]))
def test_early_exit_matches_reference(case):
    from paper_2403_09070_b200 import gp as G

    c = GOLD["cases"][case]
    kw = dict(c["cfg"])
    min_step = kw.pop("min_step", 1e-18)
    d = _design()
    cfg = G.GpConfig(seed=1, nz=GOLD["nz"], grid_nx=GOLD["grid"], grid_ny=GOLD["grid"],
                     max_iters=GOLD["max_iters"], stop_overflow=0.0, **kw)
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg)
    st = G.init_state(d, grid, cfg, rng)
    rows = []
    st, info = G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows, rng=rng, min_step=min_step)
    _check_rows(rows, c["rows"])
    _check_info(info, c["info"])
    assert info.diverged
    _check_state(st, c["state"])


def test_rotated_second_pass_matches_reference():
    from paper_2403_09070_b200 import gp as G

    r = GOLD["rotated_second_pass"]
    d = _design()
    cfg = G.GpConfig(seed=1, nz=GOLD["nz"], grid_nx=GOLD["grid"], grid_ny=GOLD["grid"],
                     max_iters=r["max_iters"], stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg)
    st = G.init_state(d, grid, cfg, rng)
    st.fillers = G.make_fillers(d, grid, rng)
    rows1 = []
    st, _ = G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows1, rng=rng)
    _check_rows(rows1, r["rows_first"])
    mids = np.flatnonzero(d.arrays().is_macro)
    st.rot = np.zeros(d.n_insts, dtype=np.int64)
    st.rot[mids] = (np.arange(len(mids)) % 3) + 1
    assert st.rot[mids].tolist() == r["rot"]
    rows = []
    st, info = G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows, rng=rng)
    _check_rows(rows, r["rows"])
    _check_info(info, r["info"])
    _check_state(st, r["state"])
