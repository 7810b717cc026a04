#!/bin/bash
# A/B over three rounds: the default libp3d.so against variants (libp3d_<v>.so)
# usage: tools/gpu_ab3.sh TAG v1 v2 ...
TAG=$1; shift
for r in 1 2 3; do for v in base "$@"; do
  if [ "$v" = base ]; then VAR=""; else VAR=$v; fi
  P3D_LIB_VARIANT=$VAR timeout 600 python bench.py --steps 32 --warmup 8 --no-cpu-baseline > gpurun_out/ab3_${TAG}_$v.log 2>&1
  tail -1 gpurun_out/ab3_${TAG}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['roofline']['stages_us']['K1_net'], d['critical_path_us']['of_which_K1'], d['critical_path_us']['density_branch_K2_K3'], d['final_row'][1])"
done; done
