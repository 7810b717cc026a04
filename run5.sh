set -x
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -8
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --precision fp32 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_net -s 5 -c 1 -o gpurun_out/prof5_net_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:line_pass -s 30 -c 6 -o gpurun_out/prof5_spec_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof5_step_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu4 $?
