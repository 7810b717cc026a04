timeout 600 python bench.py --mode batch --batch 4 --config 2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_b4.log 2>&1; echo b4 $?; tail -1 gpurun_out/bench_b4.log | cut -c1-300
timeout 600 python bench.py --precision fp32 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fp32.log 2>&1; echo fp32 $?; tail -1 gpurun_out/bench_fp32.log | cut -c1-300
timeout 600 python bench.py --mode sharded --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sh1.log 2>&1; echo sh1 $?; tail -1 gpurun_out/bench_sh1.log | cut -c1-300
