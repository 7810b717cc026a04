#!/bin/bash
# compute-sanitizer over the loop's kernels: memcheck, racecheck
# (shared-memory hazards: the scatter's u32-split atomics, staged K1 columns,
# FFT passes), synccheck and initcheck, on the smoke run (600 cells, 12 fused
# iterations + one evaluation) and a 20-iteration config-1 loop.
# usage: tools/sanitize.sh TAG
TAG=${1:-s}
CS=/usr/local/cuda/bin/compute-sanitizer
python -c 'import __graft_entry__ as g; g.build()' 2>&1 | tail -1
cat > /tmp/p3d_cfg1.py <<'PY'
import numpy as np, sys
sys.path.insert(0, ".")
from paper_2403_09070_b200 import gp as G
from paper_2403_09070_b200.synth import CONFIGS, synth_arrays
d = synth_arrays(CONFIGS[1]["spec"])
cfg = G.GpConfig(seed=1, nz=2, grid_nx=128, grid_ny=128, max_iters=20, stop_overflow=0.0)
rng = np.random.default_rng(1)
grid = G.choose_grid(d, cfg)
st = G.init_state(d, grid, cfg, rng)
rows = []
G.run_gp3d(d, st, cfg, grid=grid, iteration_log=rows, rng=rng, use_graph=False)
print("rows", len(rows), rows[-1])
PY
printf 'import sys\nsys.path.insert(0, ".")\nimport __graft_entry__ as g\ng.smoke()\n' > /tmp/p3d_smoke.py
for tool in memcheck racecheck synccheck initcheck; do
  for name in smoke cfg1; do
    timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python /tmp/p3d_$name.py \
      > gpurun_out/san_${TAG}_${tool}_${name}.log 2>&1
    echo "$tool $name rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/san_${TAG}_${tool}_${name}.log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_${TAG}_${tool}_${name}.log | tail -1)"
  done
done
