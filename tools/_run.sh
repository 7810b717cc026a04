bash tools/gpu_quick.sh sh1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --mode sharded > gpurun_out/bench_sh1_sharded.log 2>&1; echo sharded $?; tail -2 gpurun_out/bench_sh1_sharded.log | cut -c1-600
bash tools/gpu_ncu.sh it1 "advance|dens_kernel|fused|scatter|spec_|tile_|gmax0" 13 60
