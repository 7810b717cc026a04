#!/bin/bash
# A/B environment settings over three rounds.  usage: tools/gpu_env_ab3.sh TAG "ENV=.." "ENV=.." ...
TAG=$1; shift
for r in 1 2 3; do for e in "$@"; do
  env $e timeout 600 python bench.py --steps 32 --warmup 8 --no-cpu-baseline > gpurun_out/eab3_$TAG.log 2>&1
  tail -1 gpurun_out/eab3_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['value'],1), round(d['e2e']['value'],1), d['gpu_launches'], d['final_row'][1])"
done; done
