#!/bin/bash
# Full ncu capture of one GP iteration's kernels (skips the warm-up launches).
# usage: tools/gpu_ncu.sh TAG [kernel-regex] [count]
TAG=${1:-n}; KRE=${2:-"p3d"}; CNT=${3:-14}; SKIP=${4:-120}
python -c 'import __graft_entry__ as g; g.build()' 2>&1 | tail -2
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c $CNT -o gpurun_out/prof_$TAG python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_f $?
tail -3 gpurun_out/ncu_$TAG.log
