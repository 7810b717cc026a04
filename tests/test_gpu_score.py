"""Solution score on the device (evaluate_score, model.py:364-400; SURVEY 8f
rank 4) against the reference's own Score (tests/golden/score_small.json):
HPWL at 1e-12 relative (the device sums per net in a fixed tree, the
reference sequentially), HBT count exact; the SolutionError cases."""

import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_score_vs_reference():
    from paper_2403_09070_b200.score import SolutionError, evaluate_score
    from paper_2403_09070_b200.synth import SynthSpec, synth_arrays

    g = json.load(open(os.path.join(GOLD, "score_small.json")))
    d = synth_arrays(SynthSpec(**g["spec"]))
    hbt = {int(k): tuple(v) for k, v in g["hbt"].items()}
    sol = SimpleNamespace(die=np.array(g["die"]), x=np.array(g["x"]), y=np.array(g["y"]),
                          rot=np.array(g["rot"]), hbt_xy=hbt)
    sc = evaluate_score(d, sol)
    assert sc.hbt_count == g["hbt_count"]
    assert sc.hpwl == pytest.approx(g["hpwl"], rel=1e-12)
    assert sc.raw_score == pytest.approx(g["raw_score"], rel=1e-12)
    k = next(iter(hbt))
    sol.hbt_xy = {j: v for j, v in hbt.items() if j != k}  # crossing net without its HBT
    with pytest.raises(SolutionError):
        evaluate_score(d, sol)
    assert evaluate_score(d, sol, allow_illegal=True).hbt_count == g["hbt_count"] - 1
