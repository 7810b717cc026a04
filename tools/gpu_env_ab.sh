#!/bin/bash
# A/B an environment setting on the bench.  usage: tools/gpu_env_ab.sh TAG "ENV=.." "ENV=.." ...
TAG=$1; shift
for e in "" "$@" "" "$@"; do
  env $e timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/eab_$TAG.log 2>&1
  tail -1 gpurun_out/eab_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['value'],1), {k: v['ms'] for k, v in d['roofline']['per_family'].items()})"
done
