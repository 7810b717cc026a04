python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -2
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/tests_f5.log 2>&1; tail -2 gpurun_out/tests_f5.log
timeout 600 python bench.py --steps 30 --warmup 5 --cpu-seconds 20 > gpurun_out/bench_f5.log 2>&1; echo bench $?; tail -1 gpurun_out/bench_f5.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_f5_ref.log 2>&1; echo ref $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f5.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l $?
bash tools/gpu_ncu.sh f5 "advance|dens_kernel|fused|gather|scatter|spec_|tile_|gmax0" 11 60
for c in 1 2 4; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f5_c$c.log 2>&1; echo cfg$c $?; done
timeout 600 python bench.py --mode batch --batch 4 --config 2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f5_b4.log 2>&1; echo b4 $?
timeout 600 python bench.py --precision fp32 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f5_fp32.log 2>&1; echo fp32 $?
timeout 600 python bench.py --mode sharded --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f5_sh1.log 2>&1; echo sh1 $?
