"""The drop-in at the reference's own call site: place3d.flow.run_flow
(flow.py:72-165, the UNMODIFIED reference installed in baseline/_ref) with
``place3d.gp.run_gp3d`` / ``run_gp2d_multi`` swapped for the device loops.
Rotation MILP, legalization, HBT insertion, detailed placement and scoring
stay the reference's host code, exactly as INTEGRATION.md §1 describes.

Golden: tests/golden/flow_small.json, the same flows run by the reference
alone (make_golden.py --flow) on the reference's own end-to-end designs
(test_acceptance.py:329-360).  Gates:
  * 3D flow: every GP log row (both run_gp3d passes, the second with the
    MILP-rotated macro) within 1e-6 of the reference, and the flow's scored
    HPWL within the north_star's 0.5% with the same HBT count (measured:
    identical score, rows within 1.5e-7 after 861 iterations);
  * 2D flow: the first pass as above; the run_gp2d_multi pass ends inside the
    reference's own 1e-15-perturbation band (tests/golden/flow_small.json).
"""

import json
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "flow_small.json")))


@pytest.fixture(scope="module")
def place3d():
    if not os.path.isdir(os.path.join(REF, "place3d")):
        pytest.skip("baseline/_ref (the installed reference) is absent")
    sys.path.insert(0, REF)
    try:
        import place3d.flow  # noqa: F401
        import place3d.gp
        import place3d.synth
    finally:
        sys.path.remove(REF)
    return sys.modules["place3d"]


@pytest.mark.parametrize("name", ["flow3d", "flow2d"])
def test_run_flow_with_device_gp(place3d, name, monkeypatch):
    from paper_2403_09070_b200 import gp as G
    from paper_2403_09070_b200 import gp2d as G2

    gpm = place3d.gp
    calls, n_first = [], []

    def gp3d(*a, **k):
        calls.append("gp3d")
        out = G.run_gp3d(*a, **k)
        n_first.append(len(k["iteration_log"]))
        return out

    def gp2d(*a, **k):
        calls.append("gp2d")
        return G2.run_gp2d_multi(*a, **k)

    monkeypatch.setattr(gpm, "run_gp3d", gp3d)
    monkeypatch.setattr(gpm, "run_gp2d_multi", gp2d)
    g = GOLD[name]
    from place3d.model import parse_design
    from place3d.synth import SynthSpec, gen_synthetic

    d = parse_design(gen_synthetic(SynthSpec(**g["spec"])))
    sol, rep, rows, _ = place3d.flow.run_flow(d, gpm.GpConfig(seed=1, max_iters=g["max_iters"]))
    assert calls == ["gp3d", "gp3d" if g["flow_path"] == "3d" else "gp2d"]
    assert rep.flow_path == g["flow_path"]
    assert rep.rotation["rotated"] == g["rotation"]["rotated"]
    got = np.array(rows, dtype=float)
    ref = np.array(g["rows"], dtype=float)
    n1 = n_first[0]
    # first pass (run_gp3d, every flow): the log rows track the reference
    # (measured <= 1.5e-7 after 500 iterations of this 8x8x8-bin design)
    assert np.array_equal(got[:n1, 0], ref[:n1, 0]) and np.array_equal(got[:n1, 2], ref[:n1, 2])
    assert np.all(np.abs(got[:n1, 1] - ref[:n1, 1]) <= 1e-6 * ref[:n1, 1])
    assert np.all(np.abs(got[:n1, 3] - ref[:n1, 3]) <= 1e-6 * np.maximum(ref[:n1, 3], 1e-3))
    if g["flow_path"] == "3d":
        # second run_gp3d pass with the MILP-rotated macro, then the
        # reference's legalization / DP / scoring: same rows, same score
        assert got.shape == ref.shape
        assert np.all(np.abs(got[:, 1] - ref[:, 1]) <= 1e-6 * ref[:, 1])
        assert rep.final_overflow == pytest.approx(g["final_overflow"], rel=1e-6)
        assert abs(rep.hpwl - g["hpwl"]) <= 5e-3 * g["hpwl"], (rep.hpwl, g["hpwl"])
        assert rep.hbt_count == g["hbt_count"]
    else:
        # run_gp2d_multi is chaotic on this 120-cell design: the reference's
        # own end state under 1e-15 relative perturbations of the density
        # force (make_golden.py --flow, 24 seeds) spans HPWL 20,556-30,109
        # (-8% / +35% of the unperturbed 22,262.5): no implementation that is
        # not bit-identical to numpy can be held closer than that band.
        # Gate: inside the band widened by 5%, with the same HBT count.
        ends = [{**g, "n_rows": len(g["rows"])}] + g["band"]
        lo = min(e["hpwl"] for e in ends) * (1 - 5e-2)
        hi = max(e["hpwl"] for e in ends) * (1 + 5e-2)
        assert lo <= rep.hpwl <= hi, (rep.hpwl, lo, hi)
        assert rep.hbt_count in {e["hbt_count"] for e in ends}
        # the stop iteration itself is chaotic (923-1,000 rows in the band, and
        # shorter runs when overflow dips under the stop threshold earlier):
        # the run either converged or used its whole budget
        n2 = len(rows) - n1
        assert rep.final_overflow <= 0.10 or n2 == g["max_iters"], (rep.final_overflow, n2)
    print(f"{name}: hpwl {rep.hpwl} vs {g['hpwl']}, hbts {rep.hbt_count} vs {g['hbt_count']}")
