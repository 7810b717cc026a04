"""Golden fixture for the multi-die 2D GP (run_gp2d_multi, gp.py:531-690;
SURVEY 8f rank 1) from the REFERENCE itself (run in the build container):

    python tests/golden/make_gp2d.py

A 2,000-instance design is placed by a short 3D run first (so the partition
has crossing nets), then run_gp2d_multi runs max_iters iterations; the fixture
holds the 3D end state (input), the log rows, the final x, y and the HBT
centres.  The reference is never imported at test time or on the GPU box.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from place3d import gp as rgp  # noqa: E402
from place3d.model import parse_design  # noqa: E402
from place3d.synth import SynthSpec, gen_synthetic  # noqa: E402

SPEC = dict(n_insts=2000, n_macros=6, r_ma=0.30, seed=3, nets_per_inst=1.2)


VARIANTS = [  # python make_gp2d.py --variants -> gp2d_variants.json
    dict(n_insts=2000, n_macros=6, r_ma=0.55, seed=5, nets_per_inst=1.2),
    dict(n_insts=3000, n_macros=12, r_ma=0.30, seed=6, nets_per_inst=1.3),
]


def run_case(spec):
    d = parse_design(gen_synthetic(SynthSpec(**spec)))
    cfg3 = rgp.GpConfig(seed=1, nz=2, grid_nx=32, grid_ny=32, max_iters=40, stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = rgp.choose_grid(d, cfg3)
    st = rgp.init_state(d, grid, cfg3, rng)
    st, _ = rgp.run_gp3d(d, st, cfg3, grid=grid, rng=rng)
    x0, y0, z0, rot, dz = st.x.copy(), st.y.copy(), st.z.copy(), np.asarray(st.rot).copy(), st.dz
    cfg = rgp.GpConfig(seed=1, max_iters=30, stop_overflow=0.0)
    rows = []
    st, info, hbts = rgp.run_gp2d_multi(d, st, cfg, iteration_log=rows,
                                        rng=np.random.default_rng(5))
    return dict(spec=spec, max_iters=30, stop_overflow=0.0, rng_seed=5, dz=float(dz),
                x0=x0.tolist(), y0=y0.tolist(), z0=z0.tolist(), rot=rot.tolist(),
                rows=[list(map(float, r)) for r in rows], x=st.x.tolist(), y=st.y.tolist(),
                iterations=info.iterations, final_overflow=info.final_overflow,
                hbts={str(k): list(v) for k, v in hbts.items()})


def variants():
    out = [run_case(spec) for spec in VARIANTS]
    with open(os.path.join(HERE, "gp2d_variants.json"), "w") as fh:
        json.dump(out, fh)
    for c in out:
        print(c["spec"], c["rows"][-1], len(c["hbts"]))


def main():
    d = parse_design(gen_synthetic(SynthSpec(**SPEC)))
    cfg3 = rgp.GpConfig(seed=1, nz=2, grid_nx=32, grid_ny=32, max_iters=40, stop_overflow=0.0)
    rng = np.random.default_rng(1)
    grid = rgp.choose_grid(d, cfg3)
    st = rgp.init_state(d, grid, cfg3, rng)
    st, _ = rgp.run_gp3d(d, st, cfg3, grid=grid, rng=rng)
    x0, y0, z0, rot, dz = st.x.copy(), st.y.copy(), st.z.copy(), np.asarray(st.rot).copy(), st.dz
    cfg = rgp.GpConfig(seed=1, max_iters=30, stop_overflow=0.0)
    rows = []
    st, info, hbts = rgp.run_gp2d_multi(d, st, cfg, iteration_log=rows,
                                        rng=np.random.default_rng(5))
    out = dict(spec=SPEC, max_iters=30, stop_overflow=0.0, rng_seed=5, dz=float(dz),
               x0=x0.tolist(), y0=y0.tolist(), z0=z0.tolist(), rot=rot.tolist(),
               rows=[list(map(float, r)) for r in rows], x=st.x.tolist(), y=st.y.tolist(),
               iterations=info.iterations, final_overflow=info.final_overflow,
               hbts={str(k): list(v) for k, v in hbts.items()})
    with open(os.path.join(HERE, "gp2d_small.json"), "w") as fh:
        json.dump(out, fh)
    print(len(rows), rows[-1], len(hbts))


if __name__ == "__main__":
    variants() if "--variants" in sys.argv else main()
