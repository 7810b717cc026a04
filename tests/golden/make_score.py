"""Golden fixture for the solution score (evaluate_score, model.py:364-400;
SURVEY 8f rank 4) from the REFERENCE itself (run in the build container):

    python tests/golden/make_score.py

A synthetic design gets a random solution (die, lower-left x/y, rotation, one
HBT per crossing net); the fixture holds the solution and the reference's
Score.  The reference is never imported at test time or on the GPU box.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from place3d.model import Solution, evaluate_score, parse_design  # noqa: E402
from place3d.synth import SynthSpec, gen_synthetic  # noqa: E402

SPEC = dict(n_insts=2000, n_macros=6, r_ma=0.30, seed=3, nets_per_inst=1.2)


def main():
    d = parse_design(gen_synthetic(SynthSpec(**SPEC)))
    rng = np.random.default_rng(8)
    n = len(d.insts)
    die = rng.integers(0, 2, n).astype(np.int8)
    x = rng.uniform(0, d.die.width * 0.9, n)
    y = rng.uniform(0, d.die.height * 0.9, n)
    rot = rng.integers(0, 4, n)
    hbt = {}
    for net in d.nets:
        dies = {int(die[i]) for i, _ in net.pins}
        if len(dies) == 2:
            hbt[net.index] = (float(rng.uniform(0, d.die.width)), float(rng.uniform(0, d.die.height)))
    sol = Solution(die=die, x=x, y=y, rot=rot, hbt_xy=hbt)
    sc = evaluate_score(d, sol)
    out = dict(spec=SPEC, die=die.tolist(), x=x.tolist(), y=y.tolist(), rot=rot.tolist(),
               hbt={str(k): list(v) for k, v in hbt.items()}, hpwl=sc.hpwl,
               hbt_count=sc.hbt_count, raw_score=sc.raw_score)
    with open(os.path.join(HERE, "score_small.json"), "w") as fh:
        json.dump(out, fh)
    print(sc)


if __name__ == "__main__":
    main()
