#!/bin/bash
# A/B environment settings on the bench, printing it/s and the overlapped critical path.
# usage: tools/gpu_env_crit.sh TAG "ENV=.." ...
TAG=$1; shift
for e in "" "$@" "" "$@"; do
  env $e timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ecrit_$TAG.log 2>&1
  tail -1 gpurun_out/ecrit_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['value'],1), d.get('critical_path_us'))"
done
