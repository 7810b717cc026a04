#!/bin/bash
# The bench lines of the evidence run (no profiling): config 3 headline (with
# the CPU baseline), configs 1 / 2 / 4, the config-5-style batch, sharded
# world 1.  usage: tools/gpu_benches.sh TAG
TAG=${1:-b}
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-seconds 20 > gpurun_out/bench_$TAG.log 2>&1; echo bench $?
for c in 1 2 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$c.log 2>&1; echo cfg$c $?; done
timeout 900 python bench.py --mode batch --batch 4 --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_b4.log 2>&1; echo b4 $?
timeout 900 python bench.py --mode sharded --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_sh1.log 2>&1; echo sh1 $?
