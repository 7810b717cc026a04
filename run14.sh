set -x
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches14_cfg3.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu4 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spec_|fused_net" -s 30 -c 4 -o gpurun_out/prof14 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 $?
