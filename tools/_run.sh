python -c 'import __graft_entry__ as g; g.build()' >/dev/null 2>&1
export P3D_BENCH_DEVICE=0 P3D_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --config 2 > gpurun_out/b2_sharded.log 2>&1; echo sharded $?
tail -1 gpurun_out/b2_sharded.log | cut -c1-700
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --config 2 --mode replicas > gpurun_out/b2_rep.log 2>&1; echo replicas $?
tail -1 gpurun_out/b2_rep.log | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 2 --warmup 1 --impl reference --config 1 > gpurun_out/b2_ref.log 2>&1; echo ref $?
tail -1 gpurun_out/b2_ref.log | cut -c1-300
