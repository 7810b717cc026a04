#!/bin/bash
# ncu --set full (source-correlated) capture of one steady iteration's K4 / K5b
TAG=${1:-tail}
python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dens_kernel|advance_kernel" -s 40 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_f $?
