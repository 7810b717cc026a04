set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scatter_cells -s 25 -c 1 -o gpurun_out/prof7_scatter_it25 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dens_kernel -s 25 -c 1 -o gpurun_out/prof7_dens_it25 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spec_ -s 15 -c 3 -o gpurun_out/prof7_spec python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu3 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7_cfg3.csv python bench.py --steps 10 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu4 $?
