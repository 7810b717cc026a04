"""Post-GP steps on the device against runs of the reference itself
(tests/golden/make_golden.py --rebalance / --check):

* legalize.rebalance_partition (legalize.py:464-499): the same instances move
  to the same die planes, or the same LegalizationError message, on partitions
  that need many moves, a GP result, caps that force moves both ways, and caps
  no partition meets;
* check.check_solution (check.py:74-152): the same violations (messages
  identical; overlap / spacing pairs compared as sets, the reference lists
  them in hash-bucket order), pass flag and score, on legal flow outputs and
  deliberately broken copies (moved, rotated, stacked and out-of-die cells;
  missing, extra, stacked and out-of-die terminals; all cells on one die).
"""

import dataclasses
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _design(spec):
    from paper_2403_09070_b200.synth import SynthSpec, synth_arrays

    return synth_arrays(SynthSpec(**spec))


@pytest.mark.parametrize("name", ["small", "cfg1"])
def test_rebalance_partition_vs_reference(name):
    from paper_2403_09070_b200.legalize import LegalizationError, rebalance_partition
    from paper_2403_09070_b200.model import PlacementState

    g = json.load(open(os.path.join(GOLD, "rebalance.json")))[name]
    d0 = _design(g["spec"])
    n, dz = d0.n_insts, g["dz"]
    rot = np.array(g["rot"])
    top, bot = np.full(n, 3 * dz / 4), np.full(n, dz / 4)
    zs = {"all_top": (top, 0), "all_bottom": (bot, 0), "all_top_rotated": (top, 1),
          "gp": (np.array(g["z_gp"]), 0), "gp_tight_top": (np.array(g["z_gp"]), 1),
          "alternating": (np.where(np.arange(n) % 3 == 0, dz / 4, 3 * dz / 4), 1),
          "both_ways": (top, 0), "tight_caps": (top, 0)}
    for cname, ref in g["cases"].items():
        z, use_rot = zs[cname]
        d = _design(g["spec"])
        ut, ub = ref["caps"]
        if ut is not None or ub is not None:
            d.die = dataclasses.replace(
                d.die, max_util_top=ut if ut is not None else d.die.max_util_top,
                max_util_bottom=ub if ub is not None else d.die.max_util_bottom)
        st = PlacementState(x=np.zeros(n), y=np.zeros(n), z=z.copy(),
                            rot=rot.copy() if use_rot else np.zeros(n, dtype=np.int64), dz=dz)
        if ref["ok"]:
            rebalance_partition(d, st)
            moved = np.flatnonzero(st.z != z)
            assert moved.tolist() == ref["moved"], cname
            assert st.z[moved].tolist() == ref["z_moved"], cname
        else:
            with pytest.raises(LegalizationError) as e:
                rebalance_partition(d, st)
            assert str(e.value) == ref["error"], cname


@pytest.mark.parametrize("name", ["flow3d", "flow2d"])
def test_check_solution_vs_reference(name):
    from paper_2403_09070_b200.check import check_solution

    g = json.load(open(os.path.join(GOLD, "check.json")))[name]
    d = _design(g["spec"])

    class Sol:
        pass

    for cname, ref in g["cases"].items():
        c = ref["solution"]
        s = Sol()
        s.die, s.rot = np.array(c["die"]), np.array(c["rot"])
        s.x, s.y = np.array(c["x"], float), np.array(c["y"], float)
        s.hbt_xy = {int(k): tuple(v) for k, v in c["hbt_xy"].items()}
        rep = check_solution(d, s)
        assert rep.passed == ref["passed"], cname
        got = [str(v) for v in rep.violations]
        assert sorted(got) == sorted(ref["violations"]), (cname, got[:5], ref["violations"][:5])
        # the reference's order outside the pair searches
        pairs = ("[overlap]", "[hbt-spacing]")
        assert [v for v in got if not v.startswith(pairs)] == \
            [v for v in ref["violations"] if not v.startswith(pairs)], cname
        assert rep.hpwl == pytest.approx(ref["hpwl"], rel=1e-12)
        assert rep.hbt_count == ref["hbt_count"]
        assert rep.raw_score == pytest.approx(ref["raw_score"], rel=1e-12)


@pytest.mark.parametrize("rotated", [False, True])
def test_optimal_hbt_centers_vs_oracle(rotated):
    """wirelength.optimal_hbt_centers (wirelength.py:325-342)
    against the oracle's restatement (oracle.port.hbt_centers, pinned to the
    reference by test_oracle.py) on a config-1 design with random positions
    across both dies (and quarter-turned instances): the same crossing nets,
    the same centres bit for bit."""
    from oracle import port as P
    from paper_2403_09070_b200 import wirelength as wl
    from paper_2403_09070_b200.synth import CONFIGS, synth_arrays

    d = synth_arrays(CONFIGS[1]["spec"])
    a = d.arrays()
    rng = np.random.default_rng(5)
    dz = 47.52
    x = rng.uniform(0, d.die.width, a.n_inst)
    y = rng.uniform(0, d.die.height, a.n_inst)
    z = np.where(rng.random(a.n_inst) < 0.5, dz / 4, 3 * dz / 4)
    rot = rng.integers(0, 4, a.n_inst) if rotated else np.zeros(a.n_inst, dtype=np.int64)
    got = wl.optimal_hbt_centers(a, x, y, z, rot, dz)
    want = P.hbt_centers(a, x, y, z, rot, dz)
    assert len(want) > 1000 and got.keys() == want.keys()
    assert all(got[j] == want[j] for j in want)
