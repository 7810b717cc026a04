#!/bin/bash
# A/B library variants on the bench with the overlapped critical path.
# usage: tools/gpu_ab_crit.sh TAG v1 v2 ...   ("base" = the default library)
TAG=$1; shift
for v in base "$@" base "$@"; do
  if [ "$v" = base ]; then VAR=""; else VAR=$v; fi
  P3D_LIB_VARIANT=$VAR timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/abc_${TAG}_$v.log 2>&1
  tail -1 gpurun_out/abc_${TAG}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), {k: v['ms'] for k, v in d['roofline']['per_family'].items()}, d.get('critical_path_us'))"
done
