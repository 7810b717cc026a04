"""Per-rank, per-iteration exchange bytes of the sharded loop at a config:
halo mode (partition.HaloPlan on the locality order) vs the round-robin
mode's owner-sum reduce-scatter + pos4 all-gather; plus the rho all-reduce
both modes share (the numbering runs on the GPU when there is one).  usage: python tools/halo_bytes.py CONFIG"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_09070_b200.partition import HaloPlan, locality_order  # noqa: E402
from paper_2403_09070_b200.synth import CONFIGS, cached_synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = CONFIGS[cfg]
d = cached_synth(c["spec"])
a = d.arrays()
I = d.n_insts
t0 = time.time()
perm = locality_order(a.net_ptr, a.pin_inst, I)
t_order = time.time() - t0
inv = np.empty_like(perm)
inv[perm] = np.arange(I)
rho = 8 * c["grid"] * c["grid"] * 2
out = {"config": cfg, "n_inst": I, "n_net": int(a.n_net), "order_s": round(t_order, 1), "worlds": {}}
for R in (2, 4, 8):
    slab = -(-I // R)
    pl = HaloPlan(a.net_ptr, inv[a.pin_inst], I, R, slab)
    halo = [pl.exchange_bytes(r) for r in range(R)]
    dup = sum(int(pl.touches[r].sum()) for r in range(R)) / a.n_net
    rr = 2 * 32 * slab * R
    out["worlds"][R] = {"halo_positions_max_MB": max(halo) / 1e6, "round_robin_MB": rr / 1e6,
                        "rho_allreduce_MB": rho / 1e6,
                        "ratio_data_path": (max(halo) + rho) / (rr + rho),
                        "net_evaluations_per_net": round(dup, 3)}
print(json.dumps(out), flush=True)
