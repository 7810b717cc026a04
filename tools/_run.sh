python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
( time timeout 1500 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline ) > gpurun_out/bench_cfg4.log 2>&1; echo rc $?
tail -5 gpurun_out/bench_cfg4.log | cut -c1-1500
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --mode sharded > gpurun_out/bench_cfg4_sh.log 2>&1; echo rc $?; tail -1 gpurun_out/bench_cfg4_sh.log | cut -c1-400
