"""Break the bench's end-to-end region into its parts (H2D, init, K steps with
per-step row reads, D2H) with CUDA events.  usage: python tools/e2e_probe.py [K]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2403_09070_b200 import gp as G  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
design, grid_n, spec = bench.setup_design(3, 0)
cfg, grid, st, pos0 = bench.make_problem_inputs(design, spec, grid_n, 200, G)
prob = G.Gp3dProblem(design, grid, st.fillers, cfg, st.rot)
prob.init_loop(pos0)
graph = prob.capture(1)
for _ in range(5):
    graph.replay()
torch.cuda.synchronize()
host_pos = torch.from_numpy(pos0).pin_memory()
host_row = torch.empty(4, dtype=torch.float64).pin_memory()
host_out = torch.empty((prob.n_obj, 3), dtype=torch.float64).pin_memory()
dev_pos = torch.empty((prob.n_obj, 3), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record(s)
    dev_pos.copy_(host_pos, non_blocking=True)
    ev[1].record(s)
    prob.init_loop(dev_pos)
    ev[2].record(s)
    for k in range(K):
        graph.replay()
        host_row.copy_(prob.t_log[4 * k: 4 * k + 4], non_blocking=True)
    ev[3].record(s)
    out = prob._aos(prob.t_u)
    ev[4].record(s)
    host_out.copy_(out, non_blocking=True)
    ev[5].record(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    names = ["h2d", "init_loop", f"{K} steps", "aos", "d2h"]
    print({n: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, n in enumerate(names)},
          "total", round(ev[0].elapsed_time(ev[5]), 3), "host enqueue ms", round((t1 - t0) * 1e3, 3),
          "wall", round((t2 - t0) * 1e3, 3))
