"""Measurement of the SURVEY 8f rows built this round (GP2D, solution score)
on the GPU next to the oracle on the host (one core).  Prints JSON lines.

    python tools/bench_next.py [--config 2] [--iters 20]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--post", type=int, default=None, help="(separate mode) post-GP rows")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    args = ap.parse_args()
    import torch
    from threadpoolctl import threadpool_limits

    from oracle import port as P
    from paper_2403_09070_b200 import gp as G
    from paper_2403_09070_b200 import gp2d as G2
    from paper_2403_09070_b200.score import evaluate_score
    from paper_2403_09070_b200.synth import CONFIGS, cached_synth

    c = CONFIGS[args.config]
    d = cached_synth(c["spec"])
    # ---- GP2D: a short 3D run gives the partition, then timed 2D iterations
    cfg3 = G.GpConfig(seed=1, nz=2, grid_nx=c["grid"], grid_ny=c["grid"], max_iters=30,
                      stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = G.choose_grid(d, cfg3)
    st = G.init_state(d, grid, cfg3, rng)
    st, _ = G.run_gp3d(d, st, cfg3, grid=grid, rng=rng)
    x0, y0, z0, rot, dz = st.x.copy(), st.y.copy(), st.z.copy(), np.asarray(st.rot).copy(), st.dz
    # device-timed: one captured iteration replayed (the loop keeps going: a
    # long schedule, stop_overflow 0), CUDA events around `iters` replays
    W, K = 3, args.iters
    cfg = G.GpConfig(seed=1, max_iters=200, stop_overflow=0.0)
    t0 = time.perf_counter()
    loop, pos0 = G2.setup_gp2d(d, G.PlacementState(x=x0.copy(), y=y0.copy(), z=z0.copy(),
                                                   rot=rot, dz=dz), cfg, np.random.default_rng(5))
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    loop.init(pos0)
    loop.iterate()
    loop.init(pos0)
    graph = loop.capture()
    for _ in range(W):
        graph.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(K):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    st = loop.state()
    assert not st.done and st.it == W + K, (st.it, st.done)
    gpu_it = K / (e0.elapsed_time(e1) / 1000.0)
    ocfg = P.Cfg(seed=1, max_iters=args.iters, stop_overflow=0.0)
    orows = []
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        n_cpu = max(1, min(args.iters, 3))
        P.gp2d_run(d, x0, y0, z0, rot, dz, P.Cfg(seed=1, max_iters=n_cpu, stop_overflow=0.0),
                   np.random.default_rng(5), log=orows)
        cpu_it = n_cpu / (time.perf_counter() - t0)
    print(json.dumps({"row": "gp2d (run_gp2d_multi, gp.py:531-690)", "config": args.config,
                      "n_inst": d.n_insts, "gpu_it_s": gpu_it, "gpu_setup_s": t_setup,
                      "gpu": "device-resident loop, one CUDA graph per iteration, CUDA events",
                      "cpu_it_s": cpu_it,
                      "cpu": "oracle.port.gp2d_run, 1 thread, %d iterations" % n_cpu,
                      "note": "CPU sample uses a 3-iteration schedule (same per-iteration work)"}),
          flush=True)
    # ---- solution score on a random legal-shaped solution
    rs = np.random.default_rng(8)
    n = d.n_insts
    a = d.arrays()
    die = rs.integers(0, 2, n)
    sol_x = rs.uniform(0, d.die.width * 0.9, n)
    sol_y = rs.uniform(0, d.die.height * 0.9, n)
    srot = rs.integers(0, 4, n)
    pdie = die[a.pin_inst]
    mx = np.zeros(a.n_net, int)
    mn = np.ones(a.n_net, int)
    np.maximum.at(mx, a.pin_net, pdie)
    np.minimum.at(mn, a.pin_net, pdie)
    hbt = {int(j): (float(rs.uniform(0, d.die.width)), float(rs.uniform(0, d.die.height)))
           for j in np.flatnonzero(mx > mn)}

    class Sol:
        pass

    sol = Sol()
    sol.die, sol.x, sol.y, sol.rot, sol.hbt_xy = die, sol_x, sol_y, srot, hbt
    evaluate_score(d, sol)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k = 10
    for _ in range(k):
        sc = evaluate_score(d, sol)
    gpu_s = (time.perf_counter() - t0) / k
    t0 = time.perf_counter()
    h, cnt, _ = P.score(a, d.hbt.pitch, d.hbt.cost, die, sol_x, sol_y, srot, hbt)
    cpu_s = time.perf_counter() - t0
    print(json.dumps({"row": "evaluate_score (model.py:364-400)", "config": args.config,
                      "n_net": a.n_net, "gpu_ms": gpu_s * 1e3, "cpu_ms": cpu_s * 1e3,
                      "cpu": "oracle.port.score (per-net Python loop like the reference)",
                      "hpwl_gpu": sc.hpwl, "hpwl_cpu": h, "rel": abs(sc.hpwl - h) / h}),
          flush=True)


if __name__ == "__main__" and "--post" not in sys.argv:
    main()


def post_rows(config=2):
    """rebalance_partition and check_solution on the device at `config`
    (GPU wall time around the call, synchronised)."""
    import dataclasses

    import torch

    from paper_2403_09070_b200.check import check_solution
    from paper_2403_09070_b200.legalize import rebalance_partition
    from paper_2403_09070_b200.model import PlacementState
    from paper_2403_09070_b200.synth import CONFIGS, cached_synth

    d = cached_synth(CONFIGS[config]["spec"])
    n = d.n_insts
    d.die = dataclasses.replace(d.die, max_util_top=0.45)
    dz = 100.0
    for rep in range(2):
        st = PlacementState(x=np.zeros(n), y=np.zeros(n), z=np.full(n, 75.0),
                            rot=np.zeros(n, dtype=np.int64), dz=dz)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rebalance_partition(d, st)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    moved = int((st.z != 75.0).sum())
    print(json.dumps({"row": "rebalance_partition (legalize.py:464-499)", "config": config,
                      "n_inst": n, "moves": moved, "gpu_ms": dt * 1e3,
                      "note": "all instances start on the top die, top cap 0.45"}), flush=True)
    # a legal-shaped row-aligned solution: cells on rows / sites, terminals for crossing nets
    rs = np.random.default_rng(2)
    a = d.arrays()
    die = rs.integers(0, 2, n)
    rh = np.where(die == 1, d.die.row_height_top, d.die.row_height_bottom)
    x = np.floor(rs.uniform(0, d.die.width - 2000, n))
    y = np.floor(rs.uniform(0, d.die.height - 2000, n) / rh) * rh
    pdie = die[a.pin_inst]
    mx = np.zeros(a.n_net, int)
    mn = np.ones(a.n_net, int)
    np.maximum.at(mx, a.pin_net, pdie)
    np.minimum.at(mn, a.pin_net, pdie)
    hbt = {int(j): (float(rs.uniform(0, d.die.width - 50)), float(rs.uniform(0, d.die.height - 50)))
           for j in np.flatnonzero(mx > mn)}

    class Sol:
        pass

    sol = Sol()
    sol.die, sol.x, sol.y, sol.rot, sol.hbt_xy = die, x, y, np.zeros(n, dtype=np.int64), hbt
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = check_solution(d, sol)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    kinds = {}
    for v in r.violations:
        kinds[v.kind] = kinds.get(v.kind, 0) + 1
    print(json.dumps({"row": "check_solution (check.py:74-152)", "config": config, "n_inst": n,
                      "n_net": a.n_net, "gpu_ms": dt * 1e3, "violations": kinds,
                      "note": "random row-aligned solution (overlapping): every check runs"}),
          flush=True)


if __name__ == "__main__" and "--post" in sys.argv:
    post_rows(int(sys.argv[sys.argv.index("--post") + 1]) if len(sys.argv) > sys.argv.index("--post") + 1 else 2)
