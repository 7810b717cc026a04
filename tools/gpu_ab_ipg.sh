#!/bin/bash
for r in 1 2; do
for e in "P3D_BENCH_IPG=1" "P3D_BENCH_IPG=2" "P3D_BENCH_IPG=4" "P3D_BENCH_IPG=8"; do
  env $e timeout 600 python bench.py --steps 32 --warmup 8 --no-cpu-baseline > gpurun_out/ipg.log 2>&1
  tail -1 gpurun_out/ipg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['value'],1), round(d['e2e']['value'],1), d['final_row'])"
done; done
