#!/bin/bash
TAG=k3c
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_loop.py tests/test_gpu_perop.py tests/test_gpu_shard.py -q -m gpu -x > gpurun_out/tests_$TAG.log 2>&1; tail -3 gpurun_out/tests_$TAG.log
bash tools/gpu_ab.sh $TAG old k3v2
