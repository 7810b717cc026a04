#!/bin/bash
# A/B variant libraries each with its own environment.
# usage: tools/gpu_ab_env.sh TAG "name|variant|ENV=.. ENV2=.." ...   (variant "" = default lib)
TAG=$1; shift
for rep in 1 2; do
for spec in "$@"; do
  IFS='|' read -r name var envs <<< "$spec"
  env P3D_LIB_VARIANT=$var $envs timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abe_${TAG}_$name.log 2>&1
  tail -1 gpurun_out/abe_${TAG}_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: v['ms'] for k, v in d['roofline']['per_family'].items()}, d['final_row'][1], d.get('critical_path_us'))"
done; done
