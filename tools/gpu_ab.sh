#!/bin/bash
# A/B the default libp3d.so against variant builds (libp3d_<v>.so) on the bench.
# usage: tools/gpu_ab.sh TAG v1 v2 ...   ("base" = the default library)
TAG=$1; shift
for v in base "$@" base "$@"; do
  if [ "$v" = base ]; then VAR=""; else VAR=$v; fi
  P3D_LIB_VARIANT=$VAR timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}_$v.log 2>&1
  tail -1 gpurun_out/ab_${TAG}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), {k: v['ms'] for k, v in d['roofline']['per_family'].items()}, d['final_row'][1])"
done
