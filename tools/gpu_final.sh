#!/bin/bash
# The round's evidence run on one GPU: smoke, GPU tests, the bench (with the
# CPU baseline), the reference arm, the ncu launch list, one ncu --set full
# capture of an iteration's kernels (summary + traffic json), config 1/2/4 and
# batch bench lines, GP2D / post-GP rows, and compute-sanitizer.
# usage: tools/gpu_final.sh TAG
TAG=${1:-f}
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/tests_$TAG.log 2>&1; tail -1 gpurun_out/tests_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 --cpu-seconds 20 > gpurun_out/bench_$TAG.log 2>&1; echo bench $?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_ref.log 2>&1; echo ref $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l $?
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launch_summary_$TAG.txt 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fused_net|gather_warp|tile_|scatter_tiled|spec_|dens_kernel|gmax0|advance" -s 110 -c 12 -o gpurun_out/prof_$TAG python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_f $?
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > gpurun_out/ncu_summary_$TAG.txt 2>&1
python tools/ncu_traffic.py gpurun_out/prof_$TAG.ncu-rep 3 > gpurun_out/ncu_traffic_$TAG.txt 2>&1; cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_$TAG.json 2>/dev/null
for c in 1 2 4; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$c.log 2>&1; echo cfg$c $?; done
timeout 900 python bench.py --mode batch --batch 4 --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_b4.log 2>&1; echo b4 $?
timeout 900 python bench.py --mode sharded --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_sh1.log 2>&1; echo sh1 $?
timeout 900 python tools/bench_next.py --config 2 --iters 50 > gpurun_out/next_$TAG.jsonl 2>&1; echo next $?
timeout 900 python tools/bench_next.py --post 3 >> gpurun_out/next_$TAG.jsonl 2>&1; echo post $?
# (compute-sanitizer: closed on this pool late in round 2; profiles/round2_sanitize.txt holds the last run)
