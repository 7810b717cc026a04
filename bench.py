"""GP inner-loop benchmark (BASELINE.json metric: GP iterations/sec at 800k
cells; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one full global-placement iteration (gp.py:386-444: WL + density +
field + preconditioner + Nesterov/BB step) on the synthetic config-3 design
(800,064 instances, 850k nets, 512x512x2 bins).  Under
torchrun (N>1) the default mode shards ONE placement over the N ranks
(paper_2403_09070_b200.shard: objects and nets per rank, int64 density map
all-reduced over NCCL; strong scaling); --mode replicas runs N independent
placements (seed 1 + rank; weak scaling).  The timed region is bracketed by
barriers and the max over ranks is reported.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    1: "cfg1: synthetic 2-die F2F, 10,008 cells (8 macros), 12,010 nets, 128x128x2 bins",
    2: "cfg2: synthetic 100,032 cells (32 macros), 110k nets, 256x256x2 bins",
    3: "cfg3: synthetic ICCAD-2023-case4-scale, 800,064 cells (64 macros), 850k nets, 512x512x2 bins",
    4: "cfg4: synthetic 4,000,128 cells (128 macros), 4.2M nets, 1024x1024x2 bins",
}
METRIC = "GP iterations/sec at 800k cells (WL+density+field+step); % HBM roofline"


def rank_env():
    from paper_2403_09070_b200.dist import rank_world

    return rank_world()


def setup_design(config, rank):
    from paper_2403_09070_b200.synth import CONFIGS, cached_synth, SynthSpec

    from paper_2403_09070_b200.dist import replica_seed

    c = CONFIGS[config]
    spec = c["spec"]
    if rank:
        spec = SynthSpec(**{**spec.__dict__, "seed": replica_seed(spec.seed, rank)})
    return cached_synth(spec), c["grid"], spec


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every 2 ms while the
    timed region runs (nvidia-smi's 100 ms floor is longer than the region)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.err = None

    def _run(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            get_r = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self.stop.is_set():
                self.rows.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), int(get_r(h))))
                time.sleep(0.002)
        except Exception as e:  # pragma: no cover - reported in the JSON line
            self.err = repr(e)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.rows and self.err is None and time.time() - t0 < 5.0:
            time.sleep(0.001)  # NVML is up and sampling before the timed region starts
        return self

    def __exit__(self, *a):
        n = len(self.rows)
        t0 = time.time()
        while len(self.rows) == n and self.err is None and time.time() - t0 < 0.05:
            time.sleep(0.0005)  # at least one sample after the region's work was enqueued
        self.stop.set()
        self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": self.err}
        reasons = sorted({name for _, r in self.rows for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": reasons,
                "samples": len(self.rows)}


def algorithmic_bytes(design, n_fill, grid_bins):
    """compulsory bytes per iteration per kernel family."""
    a = design.arrays()
    N, P, I, F, B = a.n_net, a.n_pin, a.n_inst, n_fill, grid_bins
    O = I + F
    return {
        "K1": 4 * N + 20 * P + 40 * I,
        "K2": 24 * O + 16 * I + 8 * F + 8 * B,
        "K3": 24 * B,
        "K4": 36 * O + 16 * I + 8 * F + 16 * B,
        "K5": 152 * O + 60 * I + 8 * F,
    }


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_baseline(design, grid_n, spec, seconds=20.0, max_iters=200):
    """Oracle port (numpy, 1 core) on the same workload: bounded sample of
    whole GP iterations (setup excluded)."""
    from threadpoolctl import threadpool_limits

    from oracle import port as P

    with threadpool_limits(limits=1):
        return _cpu_baseline(P, design, grid_n, spec, seconds, max_iters)


def _cpu_baseline(P, design, grid_n, spec, seconds, max_iters):
    cfg = P.Cfg(seed=spec.seed, nz=2, grid_nx=grid_n, grid_ny=grid_n, max_iters=max_iters,
                stop_overflow=0.0)
    rng = np.random.default_rng(spec.seed)
    g = P.grid_for(design, cfg)
    x, y, z, rot = P.start_state(design, g, cfg, rng)
    fill = P.fillers_for(design, g, rng)
    prob = P.Problem(design, g, fill, cfg, rot)
    n = prob.n_inst
    pos0 = np.zeros((prob.n_obj, 3))
    pos0[:n] = np.c_[x, y, z]
    pos0[n:] = np.c_[fill.x, fill.y, fill.z]
    opt = P.Nesterov(pos0, project=prob.project)
    it, t0, lam = 0, time.perf_counter(), None
    # same per-iteration body as oracle.port.run_loop, timed iteration by iteration
    prev_raw, prev_ovfl = None, float("inf")
    while True:
        gamma = P.gamma_at(g.db, it, cfg.max_iters, cfg)
        ev, ovfl, exact, nc = prob.evaluate(opt.v, lam or 0.0, gamma)
        if lam is None:
            lam = P.lam0(np.abs(ev.wl_grad).sum(), np.abs(ev.dens_grad).sum())
            ev.total = ev.wl_grad + lam * ev.dens_grad
        q = prob.cloud(opt.v).charge
        pre, _ = P.precond(ev.total, lam, q, prob.degree_obj, prob.is_macro_obj)
        pp = None
        if prev_raw is not None:
            pp, _ = P.precond(prev_raw[0] + lam * prev_raw[1], lam, prev_raw[2], prob.degree_obj,
                              prob.is_macro_obj)
        prev_raw = (ev.wl_grad, ev.dens_grad, q)
        opt.advance(pre, step_scale=g.wb, g_prev_reval=pp)
        lam *= P.mu_of(prev_ovfl, ovfl, cfg)
        prev_ovfl = ovfl
        it += 1
        el = time.perf_counter() - t0
        if el >= seconds or it >= max_iters:
            break
    return it / el, it, el


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_reference():
    """The unmodified reference package installed in baseline/_ref (pip
    --target; it travels to the GPU box with the snapshot), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "place3d")):
        return None
    sys.path.insert(0, REF_DIR)
    try:
        import place3d.gp  # noqa: F401
        import place3d.model  # noqa: F401
        import place3d.synth  # noqa: F401
    finally:
        sys.path.remove(REF_DIR)
    return sys.modules["place3d"]


class _IterClock(list):
    """iteration_log for the reference's run_gp3d: stamps every appended row
    (one row per GP iteration, gp.py:400-401) and ends the run after `stop`."""

    class Done(Exception):
        pass

    def __init__(self, warmup, steps, budget_s=240.0):
        super().__init__()
        self.warmup, self.stop, self.budget_s = warmup, warmup + steps, budget_s
        self.t = [time.perf_counter()]

    def append(self, row):
        super().append(row)
        self.t.append(time.perf_counter())
        if len(self) == self.warmup + 1:  # trim the timed sample to the budget
            dt = self.t[-1] - self.t[-2]
            self.stop = min(self.stop, self.warmup + max(3, int(self.budget_s / max(dt, 1e-9))))
        if len(self) >= self.stop:
            raise _IterClock.Done()


def run_reference(args, rank, world):
    """--impl reference: the reference's own run_gp3d (baseline/_ref, its stock
    numpy code path, gp.py:359-455) on rank 0's host cores, timed iteration
    by iteration through its iteration_log (setup excluded); without
    baseline/_ref, the oracle port.  Other ranks exit without work."""
    if rank != 0:
        return
    from paper_2403_09070_b200.synth import CONFIGS

    ref = _import_reference()
    c = CONFIGS[args.config]
    grid_n, spec = c["grid"], c["spec"]
    ncpu = os.cpu_count()
    W, K = max(args.warmup, 0), args.steps
    if ref is None:
        design, grid_n, spec = setup_design(args.config, 0)
        budget = min(60.0, 6.0 * (K + W))
        rate, iters, el = cpu_baseline(design, grid_n, spec, seconds=budget)
        kind, sample, W, K = "port", (f"{iters} GP iterations from the initial state "
                                      f"({el:.1f} s), oracle.port numpy, 1 thread"), 0, iters
    else:
        from threadpoolctl import threadpool_limits

        t0 = time.perf_counter()
        d = ref.model.parse_design(ref.synth.gen_synthetic(ref.synth.SynthSpec(**spec.__dict__)))
        setup_s = time.perf_counter() - t0
        cfg = ref.gp.GpConfig(seed=spec.seed, nz=2, grid_nx=grid_n, grid_ny=grid_n,
                              max_iters=200, stop_overflow=0.0)
        rng = np.random.default_rng(spec.seed)
        grid = ref.gp.choose_grid(d, cfg)
        st = ref.gp.init_state(d, grid, cfg, rng)
        # bounded sample: W + K iterations of the 200-iteration schedule, K
        # trimmed so the timed part stays within ~4 minutes (per-iteration cost
        # measured on the first timed iteration)
        W = max(W, 1)  # the first iteration also builds the reference's Gp3dProblem
        clock = _IterClock(W, K)
        with threadpool_limits(limits=ncpu):
            try:
                ref.gp.run_gp3d(d, st, cfg, grid=grid, iteration_log=clock, rng=rng)
            except _IterClock.Done:
                pass
        ts = np.array(clock.t)
        iters = len(ts) - 1 - W
        el = float(ts[-1] - ts[W])
        rate = iters / el
        kind = "reference"
        sample = (f"place3d.gp.run_gp3d (baseline/_ref, unmodified) on config {args.config}: "
                  f"{W} warm-up + {iters} timed iterations of the 200-iteration schedule "
                  f"({el:.1f} s timed; setup {setup_s:.0f} s excluded); numpy/scipy, "
                  f"threadpool limit {ncpu} (the reference loop is single-threaded); "
                  f"final row {list(clock[-1])}")
        K = iters
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "it/s", "n_gpus": args.gpus,
        "steps": K, "warmup": W, "ms_per_step": 1000.0 / rate,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOADS[args.config], "grid": [grid_n] * 2 + [2],
                                        "max_iters_schedule": 200},
        "cpu_baseline": {"value": rate, "unit": "it/s", "cores": 1, "kind": kind,
                         "sample": sample + f"; host has {ncpu} cpus"},
        "e2e": {"value": rate, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def parity_vs_reference(config, max_iters, row):
    """The bench's last log row against the reference's row at the same
    iteration (tests/golden/cfg3_rows.json, made by the reference itself)."""
    if config != 3 or max_iters != 200:
        return None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "cfg3_rows.json")) as fh:
            gold = json.load(fh)["sched200_first25"]
    except (OSError, ValueError, KeyError):
        return None
    it = int(row[0])
    if it >= len(gold):
        return {"iteration": it, "note": "beyond the committed reference rows"}
    r = gold[it]
    wl_rel = abs(row[1] - r[1]) / r[1]
    ov_rel = abs(row[3] - r[3]) / r[3]
    return {"iteration": it, "reference_row": r, "wl_rel": wl_rel, "overflow_rel": ov_rel,
            "crossings_equal": int(row[2]) == int(r[2]),
            "ok": bool(wl_rel <= 5e-3 and ov_rel <= 5e-3)}


def make_problem_inputs(design, spec, grid_n, max_iters, G):
    cfg = G.GpConfig(seed=spec.seed, nz=2, grid_nx=grid_n, grid_ny=grid_n, max_iters=max_iters,
                     stop_overflow=0.0)
    if os.environ.get("P3D_PROBE_SKIP"):  # timing probes drop work: keep the loop running
        cfg.divergence_window = 1 << 30
    rng = np.random.default_rng(spec.seed)
    grid = G.choose_grid(design, cfg)
    st = G.init_state(design, grid, cfg, rng)
    st.fillers = G.make_fillers(design, grid, rng)
    n = design.n_insts
    pos0 = np.zeros((n + st.fillers.count, 3))
    pos0[:n] = np.c_[st.x, st.y, st.z]
    pos0[n:] = np.c_[st.fillers.x, st.fillers.y, st.fillers.z]
    return cfg, grid, st, pos0


def roofline_of(design, n_fill, grid, stage_ms, config, shards=1):
    """Roofline of the dominant kernel family (SURVEY 8d algorithmic bytes;
    with `shards`, one rank's share: every family but the replicated K3)."""
    q = algorithmic_bytes(design, n_fill, grid.n_bins)
    q = {k: (v if k == "K3" else v / shards) for k, v in q.items()}
    fam_ms = {"K1": stage_ms[0] + stage_ms[1], "K2": stage_ms[2], "K3": stage_ms[3],
              "K4": stage_ms[4], "K5": stage_ms[5] + stage_ms[6]}
    dom = max(fam_ms, key=fam_ms.get)
    peak, peak_kind = load_peaks()
    achieved = q[dom] / (fam_ms[dom] / 1000.0) / 1e9
    names = ("K1_net", "K1b_gather", "K2_scatter", "K3_spectral", "K4_dens", "K5a_step0",
             "K5b_advance")
    stages_us = {n: round(float(v) * 1000.0, 1) for n, v in zip(names, stage_ms)}
    per_family = {k: {"ms": round(float(v), 4), "alg_MB": round(q[k] / 1e6, 2),
                      "GBs": round(q[k] / (v / 1000.0) / 1e9, 1) if v > 0 else None}
                  for k, v in fam_ms.items()}
    traffic = None
    try:  # DRAM bytes per iteration of the dominant family from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        if tr.get("config") == config:
            traffic = tr.get(dom)
    except (OSError, ValueError):
        pass
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
            "per_family": per_family,
            "stages_us": stages_us}


def run_batch(args, rank, world, local):
    """Config-5 style throughput: args.batch independent placements per GPU
    (seeds differ per placement and rank), each a CUDA graph of one iteration,
    replayed round-robin on its own stream so the GPU overlaps them."""
    import torch
    import torch.distributed as dist

    from paper_2403_09070_b200 import gp as G

    dev = int(os.environ.get("P3D_BENCH_DEVICE", local))
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("P3D_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    W, K, Bn = max(args.warmup, 3), args.steps, args.batch
    max_iters = max(200, W + 2 * K + 2)
    ipg = int(os.environ.get("P3D_BENCH_IPG", "8"))  # iterations per replay, as run_gp3d
    probs, steppers, starts = [], [], []
    for b in range(Bn):
        design, grid_n, spec = setup_design(args.config, rank * Bn + b)
        cfg, grid, st, pos0 = make_problem_inputs(design, spec, grid_n, max_iters, G)
        prob = G.Gp3dProblem(design, grid, st.fillers, cfg, st.rot, precision=args.precision)
        prob.init_loop(pos0)
        probs.append(prob)
        steppers.append(prob.stepper(ipg))  # iteration 0, then steady graphs (uploaded)
        prob.init_loop(pos0)
        steppers[-1].reset()
        starts.append(pos0)
    streams = [torch.cuda.Stream() for _ in range(Bn)]
    cur = torch.cuda.current_stream()

    def step(n):
        for s_ in streams:
            s_.wait_stream(cur)
        k = 0
        while k < n:  # one replay per placement in turn, each on its own stream
            c = min(ipg, n - k)
            for st_, s_ in zip(steppers, streams):
                with torch.cuda.stream(s_):
                    st_(c)
            k += c
        for s_ in streams:
            cur.wait_stream(s_)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    step(W)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        e0.record(cur)
        step(K)
        e1.record(cur)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    for p_ in probs:
        s_ = p_.state()
        assert not s_.done and s_.it == W + K, f"loop ended early (it={s_.it})"
    # end to end: every placement's host positions in, K steps, positions out
    host_pos = [torch.from_numpy(p0).pin_memory() for p0 in starts]
    host_out = [torch.empty((3, p_.n_obj), dtype=torch.float64).pin_memory() for p_ in probs]
    host_rows = torch.empty((Bn, K, 4), dtype=torch.float64).pin_memory()
    row_stream = torch.cuda.Stream()  # each step's rows are read back beside the next step
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    f0.record(cur)
    for p_, st_, h in zip(probs, steppers, host_pos):
        p_.init_loop(h.to("cuda", non_blocking=True))
        st_.reset()
    k = 0
    while k < K:  # the timed replays; each replay's rows read back beside the next one
        c = min(ipg, K - k)
        step(c)
        row_stream.wait_stream(cur)
        with torch.cuda.stream(row_stream):
            for b, p_ in enumerate(probs):
                host_rows[b, k:k + c].copy_(p_.t_log[4 * k: 4 * (k + c)].view(c, 4),
                                            non_blocking=True)
        k += c
    for p_, h in zip(probs, host_out):
        h.copy_(p_.t_u[: 3 * p_.n_obj].view(3, p_.n_obj), non_blocking=True)
    cur.wait_stream(row_stream)
    f1.record(cur)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    t = torch.tensor([ms, e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(t[0]), float(t[1])
    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return
    units = world * Bn * K
    line = {
        "metric": METRIC, "value": units / (ms / 1000.0), "unit": "it/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (paper_2403_09070_b200.synth, one seed per placement)",
        "config": {"workload": f"cfg5-style: {Bn} independent placements per GPU of "
                               + WORKLOADS[args.config], "placements": world * Bn,
                   "parallelism": f"{Bn} concurrent graphs per GPU x {world} GPUs",
                   "mode": "batch", "iterations_per_graph": ipg,
                   "l2": "no flush: working sets exceed L2"},
        "e2e": {"value": units / (e2e_ms / 1000.0), "unit": "it/s",
                "h2d_bytes_per_step": int(sum(h.numel() * 8 for h in host_pos) / K),
                "d2h_bytes_per_step": int(32 * Bn + sum(h.numel() * 8 for h in host_out) / K)},
        "gpu_launches": int((_lib_kernels(probs[0]) - 1) * Bn * K),  # steady iterations
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _lib_kernels(prob):
    from paper_2403_09070_b200 import _lib

    return _lib.load().p3d_gp_kernels_per_iteration(_lib.byref(prob.gp))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default=None, choices=["fused", "sharded", "replicas", "batch"],
                    help="fused: one GPU, the whole iteration in one CUDA graph (N=1 default); "
                         "sharded: ONE placement partitioned over the N ranks (N>1 default, "
                         "strong scaling); replicas: N independent placements (weak scaling); "
                         "batch: --batch independent placements per GPU, their iteration "
                         "graphs replayed on concurrent streams (config 5 throughput)")
    ap.add_argument("--batch", type=int, default=8, help="placements per GPU in --mode batch")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="WA arithmetic: fp64 numpy-order (default) or fp32 anchored")
    args = ap.parse_args()
    rank, world, local = rank_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not under torchrun: spawn one rank per GPU ourselves
        import subprocess

        port = os.environ.get("MASTER_PORT", "29511")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", port, os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    mode = args.mode or ("sharded" if world > 1 else "fused")
    if mode == "fused" and world > 1:
        mode = "replicas"
    if mode == "batch":
        return run_batch(args, rank, world, local)

    import torch
    import torch.distributed as dist

    # test hooks (not for measurements): P3D_BENCH_DEVICE pins every rank to one
    # GPU, P3D_BENCH_BACKEND=gloo replaces NCCL (several ranks on one device)
    dev = int(os.environ.get("P3D_BENCH_DEVICE", local))
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("P3D_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    from paper_2403_09070_b200 import _lib
    from paper_2403_09070_b200 import gp as G

    design, grid_n, spec = setup_design(args.config, rank if mode == "replicas" else 0)
    W, K = max(args.warmup, 3), args.steps
    max_iters = max(200, W + 2 * K + 2)
    cfg, grid, st, pos0 = make_problem_inputs(design, spec, grid_n, max_iters, G)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    ipg = 1  # iterations per graph replay in the timed region
    if mode == "sharded":
        from paper_2403_09070_b200.shard import ShardedGp3d

        runner = ShardedGp3d(design, grid, st.fillers, cfg, st.rot, precision=args.precision)
        prob = runner.prob
        step = runner.iterate
        init_loop = runner.init_loop  # caller's instance order -> the shard's numbering
        runner.init_loop(pos0)
        if runner.comm.nccl or not runner.comm.on:  # the iteration (+ collectives) as one graph
            try:  # iteration 0's graph with the initial step, then the steady-state one
                step = runner.stepper()
                ipg = 8  # ShardedGp3d.stepper: steady iterations per replay
                step(ipg + 2)  # each graph's first launch uploads it: not in the timed region
                runner.init_loop(pos0)
                step.reset()
            except Exception as exc:  # pragma: no cover - eager fallback, reported
                print(f"# sharded graph capture failed ({exc!r}); running eagerly",
                      file=sys.stderr)
                runner.init_loop(pos0)
    else:
        prob = G.Gp3dProblem(design, grid, st.fillers, cfg, st.rot, precision=args.precision)
        init_loop = prob.init_loop
        prob.init_loop(pos0)
        # as run_gp3d replays them (Gp3dProblem.run: iteration 0, then 8 steady
        # iterations per graph, so consecutive iterations keep their
        # programmatic-dependent-launch edges); the remainder of K one by one:
        # exactly K iterations.  Each graph is launched (uploaded) once before
        # the warm-up, then the loop re-initialised.
        ipg = int(os.environ.get("P3D_BENCH_IPG", "8"))
        steady = os.environ.get("P3D_BENCH_STEADY", "1") == "1"  # A/B switch
        step = prob.stepper(ipg, steady=steady)
        prob.init_loop(pos0)
        step.reset()

    # ---- device-resident timed region
    step(W)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        step(K)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    s = prob.state()
    if not os.environ.get("P3D_PROBE_SKIP"):  # timing probes drop work: no assert
        assert not s.done and s.it == W + K, f"loop ended early (it={s.it}, done={s.done})"

    # ---- per-stage attribution (fused: the same iteration captured with
    # event-record nodes between the stages, replayed K times)
    stage = np.zeros(7)
    if mode != "sharded":
        buf = (C.c_float * 7)()
        mg = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side), torch.cuda.graph(mg, stream=side):
            _lib.call("p3d_gp_iterate_marked", _lib.byref(prob.gp), _lib.stream_ptr())
        stream.wait_stream(side)
        for _ in range(K):
            mg.replay()
            torch.cuda.synchronize()
            _lib.call("p3d_gp_stage_times", buf)
            stage += np.frombuffer(buf, dtype=np.float32)
        stage /= K
        # the timed iterations are steady ones (W >= 3): no initial-step kernel
        kpi = _lib.load().p3d_gp_kernels_per_iteration(_lib.byref(prob.gp)) - (1 if steady else 0)
        # the production (overlapped) iteration's critical path, from event
        # nodes at its branch points inside a replayed graph
        crit = None
        if prob.gp.overlap:
            tb = (C.c_float * 7)()
            og = torch.cuda.CUDAGraph()
            side.wait_stream(stream)
            with torch.cuda.stream(side), torch.cuda.graph(og, stream=side):
                _lib.call("p3d_gp_iterate_marked_overlap", _lib.byref(prob.gp), _lib.stream_ptr())
            stream.wait_stream(side)
            acc = np.zeros(7)
            for _ in range(K):
                og.replay()
                torch.cuda.synchronize()
                _lib.call("p3d_gp_overlap_times", tb)
                acc += np.frombuffer(tb, dtype=np.float32)
            acc = acc / K * 1000.0
            crit = {"wl_branch_K1_K1b": round(acc[1], 1), "of_which_K1": round(acc[0], 1),
                    "density_branch_K2_K3": round(acc[3], 1), "of_which_K2": round(acc[2], 1),
                    "K4_end": round(acc[4], 1), "K5_end": round(acc[6], 1)}
    else:
        # the staged protocol adds the norm pass, its finaliser and the control
        # kernel; the steady-state graph drops the initial-step pair (+2), the
        # eager path keeps it (+4)
        kpi = _lib.load().p3d_gp_kernels_per_iteration(_lib.byref(prob.gp)) + (
            2 if hasattr(step, "reset") else 4)
        marks = []
        runner.iterate(K, marks=marks)  # eager, with events between stages
        att = runner.attribute(marks)
        stage = np.array([att.get("K1", 0.0), 0.0, att.get("K2", 0.0), att.get("K3", 0.0),
                          att.get("K4", 0.0), att.get("K5", 0.0), 0.0]) / K
        comm_ms = att.get("comm", 0.0) / K

    # ---- end to end through the public API: pinned host state in, K steps with
    # the per-iteration log row read back every step, final positions out
    host_pos = torch.from_numpy(pos0).pin_memory()
    host_rows = torch.empty((max(W, K), 4), dtype=torch.float64).pin_memory()
    host_out = torch.empty((3, prob.n_obj), dtype=torch.float64).pin_memory()  # x, y, z
    dev_pos = torch.empty((prob.n_obj, 3), dtype=torch.float64, device="cuda")
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    row_stream = torch.cuda.Stream()  # each step's row is read back beside the next step

    def e2e_pass(n):
        cur = torch.cuda.current_stream()
        dev_pos.copy_(host_pos, non_blocking=True)
        init_loop(dev_pos)
        if hasattr(step, "reset"):
            step.reset()
        k = 0
        while k < n:  # the timed region's replays; each replay's log rows (one per
            c = min(ipg, n - k)  # iteration) are read back beside the next replay
            step(c)
            row_stream.wait_stream(cur)
            with torch.cuda.stream(row_stream):
                host_rows[k:k + c].copy_(prob.t_log[4 * k: 4 * (k + c)].view(c, 4),
                                         non_blocking=True)
            k += c
        host_out.copy_(prob.t_u[: 3 * prob.n_obj].view(3, prob.n_obj), non_blocking=True)
        cur.wait_stream(row_stream)  # every row is in host memory before the pass ends

    e2e_pass(W)  # warm-up of the API path (first-use allocations, pinned staging)
    barrier()
    f0.record(stream)
    e2e_pass(K)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    barrier()

    # max over ranks
    from paper_2403_09070_b200.dist import max_over_ranks

    ms, e2e_ms = max_over_ranks([ms, e2e_ms])
    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return
    units = world * K if mode == "replicas" else K
    it_s = units / (ms / 1000.0)
    e2e_it_s = units / (e2e_ms / 1000.0)
    ws_mb = (sum(t.numel() * t.element_size() for t in prob._keep.items) +
             sum(t.numel() * t.element_size() for t in prob._dtopo.keep.items)) / 1e6
    parallelism = {"fused": "single", "replicas": f"replicas x{world}",
                   "sharded": f"sharded over {world} (instance slabs + the nets touching them "
                              f"per rank, halo positions, int64 rho all-reduce)"}[mode]
    line = {
        "metric": METRIC, "value": it_s, "unit": "it/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "weak" if mode == "replicas" else "strong",
        "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f64+f32(WA)",
        "data": "synthetic (paper_2403_09070_b200.synth == place3d.synth.gen_synthetic" +
                (", seed 1+rank)" if mode == "replicas" else ", seed 1)"),
        "config": {"workload": WORKLOADS[args.config], "n_inst": prob.n_inst,
                   "n_fill": prob.n_fill, "n_net": design.n_nets,
                   "n_pin": design.arrays().n_pin, "grid": [grid.nx, grid.ny, grid.nz],
                   "max_iters_schedule": max_iters, "parallelism": parallelism, "mode": mode,
                   "iterations_per_graph": ipg,
                   "wl_precision": args.precision,
                   "l2": f"no flush: iteration working set {ws_mb:.0f} MB > 126 MB L2"},
        "e2e": {"value": e2e_it_s, "unit": "it/s",
                "h2d_bytes_per_step": int(host_pos.numel() * 8 / K),
                "d2h_bytes_per_step": int(32 + host_out.numel() * 8 / K),
                "path": "pinned positions in, init, the K iterations as timed above with "
                        "every iteration's log row read back after its graph replay, "
                        "positions out"},
        "gpu_launches": int(kpi * K),
        "clocks": clocks.summary(),
        "final_row": list(prob.log_rows(W + K)[-1]),
    }
    line["parity"] = parity_vs_reference(args.config, max_iters, line["final_row"])
    if mode != "sharded" and crit is not None:
        line["critical_path_us"] = crit
    line["roofline"] = roofline_of(design, prob.n_fill, grid, stage, args.config,
                                   shards=world if mode == "sharded" else 1)
    if mode == "sharded":  # rank 0's stage attribution of one shard (eager replay)
        line["roofline"]["traffic"] = None
        line["roofline"]["note"] = ("rank-0 shard, eager stages; algorithmic bytes of the whole "
                                    "placement / world per family")
        line["config"]["collective_ms_per_step"] = round(comm_ms, 4)
        line["config"]["exchange_bytes_per_rank_per_step"] = runner.exchange_bytes()
        line["config"]["partition"] = ("halo: locality-ordered instance slabs, nets run on every "
                                       "rank they touch, halo positions all-to-all"
                                       if runner.halo else "round-robin K1 tasks")
    if not args.no_cpu_baseline and world == 1:
        rate, iters, el = cpu_baseline(design, grid_n, spec, seconds=args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": "it/s", "cores": 1, "kind": "port",
                                "sample": f"{iters} GP iterations of the same workload from the "
                                          f"initial state ({el:.1f} s), oracle.port numpy, 1 thread"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
