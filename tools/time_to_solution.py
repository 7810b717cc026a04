"""Time to solution of the drop-in: `gp.run_gp3d` on config 3 with the full
200-iteration schedule, wall clock through the public API (problem setup on
the host + device layouts + the graph-replayed loop + the state copied back),
with a cProfile breakdown of the host setup on stderr.  One JSON line on
stdout.  usage: python tools/time_to_solution.py [--config 3] [--profile]"""

import argparse
import cProfile
import json
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_09070_b200 import gp as G  # noqa: E402
from paper_2403_09070_b200.synth import CONFIGS, cached_synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--profile", action="store_true")
    args = ap.parse_args()
    torch.zeros(1, device="cuda")
    c = CONFIGS[args.config]
    d = cached_synth(c["spec"])
    cfg = G.GpConfig(seed=1, nz=2, grid_nx=c["grid"], grid_ny=c["grid"], max_iters=200,
                     stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg)
    st = G.init_state(d, grid, cfg, rng)
    pr = cProfile.Profile() if args.profile else None
    if pr:
        pr.enable()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = []
    st, info = G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows, rng=rng)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if pr:
        pr.disable()
        pstats.Stats(pr, stream=sys.stderr).sort_stats("cumulative").print_stats(20)
    print(json.dumps({"row": "run_gp3d time to solution", "config": args.config,
                      "iterations": info.iterations, "wall_s": t1 - t0,
                      "final_row": list(rows[-1])}))


if __name__ == "__main__":
    main()
