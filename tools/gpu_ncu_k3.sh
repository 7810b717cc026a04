#!/bin/bash
# ncu --set full (source-correlated) capture of one iteration's K3 passes
TAG=${1:-k3}
python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spec_" -s 30 -c 3 -o gpurun_out/prof_$TAG python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_f $?
tail -2 gpurun_out/ncu_$TAG.log
