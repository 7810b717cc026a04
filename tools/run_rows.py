"""Run the device GP loop on a BASELINE config and dump the log rows (json)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2403_09070_b200 import gp as G  # noqa: E402
from paper_2403_09070_b200.synth import CONFIGS, cached_synth  # noqa: E402


def main(cfg_id, precision, out, max_iters=200):
    c = CONFIGS[cfg_id]
    d = cached_synth(c["spec"])
    cfg = G.GpConfig(seed=1, nz=2, grid_nx=c["grid"], grid_ny=c["grid"], max_iters=max_iters,
                     stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg)
    st = G.init_state(d, grid, cfg, rng)
    rows = []
    G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows, rng=rng, precision=precision)
    json.dump({"config": cfg_id, "precision": precision, "max_iters": max_iters,
               "rows": [list(map(float, r)) for r in rows]}, open(out, "w"))
    print(cfg_id, precision, rows[-1])


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 200)
