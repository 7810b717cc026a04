#!/bin/bash
# One GPU round-trip: smoke, GPU parity tests, bench, launch list, full ncu of the top kernels.
# usage: tools/gpu_check.sh TAG [ncu-kernel-regex]
TAG=${1:-x}; KRE=${2:-"fused_net|dens_kernel|spec_x"}
set -x
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -2
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 15 > gpurun_out/bench_$TAG.log 2>&1; echo bench $?; tail -1 gpurun_out/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 40 -c 3 -o gpurun_out/prof_$TAG python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_f $?
