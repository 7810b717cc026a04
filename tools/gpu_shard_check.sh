#!/bin/bash
# sharded-loop check: its GPU tests, then the world-1 sharded bench line
TAG=${1:-sh}
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_loop.py -q -m gpu -x > gpurun_out/tests_$TAG.log 2>&1; tail -3 gpurun_out/tests_$TAG.log
timeout 600 python bench.py --mode sharded --steps 32 --warmup 8 --no-cpu-baseline > gpurun_out/bench_${TAG}_sh1.log 2>&1; echo sh1 $?
tail -1 gpurun_out/bench_${TAG}_sh1.log | cut -c1-400
timeout 600 python bench.py --steps 32 --warmup 8 --no-cpu-baseline > gpurun_out/bench_${TAG}.log 2>&1; echo fused $?
tail -1 gpurun_out/bench_${TAG}.log | cut -c1-400
