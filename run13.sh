timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b13.log 2>&1; echo rc $?
tail -30 gpurun_out/b13.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -3
