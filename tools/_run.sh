python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
timeout 900 python bench.py --steps 30 --warmup 5 --cpu-seconds 20 > gpurun_out/bench_final1.log 2>&1; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final1.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l $?
bash tools/gpu_ncu.sh final1 "advance|dens_kernel|fused|scatter|spec_|tile_|gmax0" 11 60
