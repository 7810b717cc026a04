set -x
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches10_cfg3.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu4 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_net -s 5 -c 1 -o gpurun_out/prof10_net python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dens_kernel -s 10 -c 1 -o gpurun_out/prof10_dens python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu3 $?
