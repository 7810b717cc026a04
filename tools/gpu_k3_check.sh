#!/bin/bash
# K3 change check: ops + loop GPU tests, A/B against libp3d_old.so, K3 ncu capture
TAG=${1:-k3}
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_loop.py tests/test_gpu_perop.py -q -m gpu -x > gpurun_out/tests_$TAG.log 2>&1; tail -3 gpurun_out/tests_$TAG.log
bash tools/gpu_ab.sh $TAG old
bash tools/gpu_ncu_k3.sh ${TAG}n
