set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap --format=csv
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
for p in fp64 fp32; do timeout 300 python tools/run_rows.py 2 $p gpurun_out/cfg2_$p.json; done
timeout 300 python tools/run_rows.py 3 fp32 gpurun_out/cfg3_fp32_20.json 20
for c in 1 2; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_net -s 5 -c 1 -o gpurun_out/prof_net_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu2 $?
ls -la gpurun_out
