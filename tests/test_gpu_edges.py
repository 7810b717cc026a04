"""run_gp3d at its boundaries, against runs of the reference itself
(tests/golden/edges.json, tests/golden/make_golden.py --edges): converged
before the first step (stop_overflow above the initial overflow), one and two
iterations (iteration 1 is the first Barzilai-Borwein step), every instance
starting on the bottom die, and a netlist of single-pin nets only (zero
wirelength and gradient: a density-only descent, gated by the reference's own
spread under 1e-12 noise on the density force).  Each case checks the log
rows, GpInfo and the returned state like test_gpu_exits.py.  (A design
without nets is outside the reference's domain: its NetBoxes raises.)"""

import json
import os

import numpy as np
import pytest

from test_gpu_exits import _check_info, _check_rows, _check_state

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "edges.json")))


def _design(nets=None):
    from paper_2403_09070_b200.model import ArrayDesign, NetlistArrays
    from paper_2403_09070_b200.synth import SynthSpec, synth_arrays

    d = synth_arrays(SynthSpec(**GOLD["spec"]))
    if nets is None:
        return d
    assert nets == "first_pin"
    a = d.arrays()
    first = a.net_ptr[:-1]
    arr = NetlistArrays(is_macro=a.is_macro, w_top=a.w_top, h_top=a.h_top, w_bot=a.w_bot,
                        h_bot=a.h_bot, net_ptr=np.arange(a.n_net + 1), pin_inst=a.pin_inst[first],
                        ox_top=a.ox_top[first], oy_top=a.oy_top[first], ox_bot=a.ox_bot[first],
                        oy_bot=a.oy_bot[first])
    return ArrayDesign(d.die, d.hbt, arr)


@pytest.mark.parametrize("name", sorted(GOLD["cases"]))
def test_edge_case_matches_reference(name):
    from paper_2403_09070_b200 import gp as G

    c = GOLD["cases"][name]
    d = _design(c["case"].get("nets"))
    cfg = G.GpConfig(seed=1, nz=GOLD["nz"], grid_nx=GOLD["grid"], grid_ny=GOLD["grid"], **c["cfg"])
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg)
    st = G.init_state(d, grid, cfg, rng)
    if c["case"].get("z") == "bottom":
        st.z[:] = grid.dz / 4
    rows = []
    st, info = G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows, rng=rng)
    if "band_wl_ovfl" in c:
        # no wirelength force: the density-only descent amplifies the int64
        # map's 2^-40 quantisation like 1e-12 relative noise on the density
        # force; the gate is the reference's own spread under that noise
        got, ref = np.array(rows, float), np.array(c["rows"], float)
        band = np.array(c["band_wl_ovfl"])
        assert got.shape == ref.shape and np.array_equal(got[:, 2], ref[:, 2])
        assert np.all(got[:, 1] == ref[:, 1])  # zero wirelength
        assert np.all(np.abs(got[:, 3] - ref[:, 3]) <= np.maximum(2 * band[:, 1], 1e-13))
        _check_info(info, c["info"], tol=1e-6)
        _check_state(st, c["state"], tol=1e-6)
        return
    _check_rows(rows, c["rows"])
    _check_info(info, c["info"])
    _check_state(st, c["state"])
