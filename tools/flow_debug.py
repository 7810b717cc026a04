"""Debug: compare the device flow's GP rows with the reference flow golden."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import place3d.flow, place3d.gp as gpm
from place3d.model import parse_design
from place3d.synth import SynthSpec, gen_synthetic
from paper_2403_09070_b200 import gp as G, gp2d as G2
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "flow_small.json")))
for name in sys.argv[1:] or ["flow3d", "flow2d"]:
    g = GOLD[name]
    d = parse_design(gen_synthetic(SynthSpec(**g["spec"])))
    cfg = gpm.GpConfig(seed=1, max_iters=g["max_iters"])
    rng = np.random.default_rng(cfg.seed)
    grid = gpm.choose_grid(d, cfg)
    st = gpm.init_state(d, grid, cfg, rng)
    rows = []
    st2, info = G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows, rng=rng)
    ref = np.array(g["rows"])
    got = np.array(rows)
    n = min(len(got), len(ref))
    rel = np.abs(got[:n, 1] - ref[:n, 1]) / ref[:n, 1]
    bad = np.flatnonzero((rel > 1e-9) | (got[:n, 2] != ref[:n, 2]))
    print(name, "grid", grid.nx, grid.ny, grid.nz, "rows", len(got), "first bad", bad[:5], rel[:5], rel.max())
    if len(bad):
        k = bad[0]
        print(" got", got[max(k-1,0):k+2].tolist(), "\n ref", ref[max(k-1,0):k+2].tolist())

print("---- full flows")
for name in sys.argv[1:] or ["flow3d", "flow2d"]:
    g = GOLD[name]
    gpm.run_gp3d, gpm.run_gp2d_multi = G.run_gp3d, G2.run_gp2d_multi
    d = parse_design(gen_synthetic(SynthSpec(**g["spec"])))
    sol, rep, rows, _ = place3d.flow.run_flow(d, gpm.GpConfig(seed=1, max_iters=g["max_iters"]))
    got, ref = np.array(rows), np.array(g["rows"])
    n = min(len(got), len(ref))
    rel = np.abs(got[:n, 1] - ref[:n, 1]) / ref[:n, 1]
    print(name, len(got), len(ref), "maxrel", rel.max(), "first>1e-6", np.flatnonzero(rel > 1e-6)[:3],
          "hpwl", rep.hpwl, g["hpwl"], "hbt", rep.hbt_count, g["hbt_count"], "ovfl", rep.final_overflow,
          g["final_overflow"], "rot", rep.rotation, g["rotation"])
