#!/bin/bash
# default bench line + sharded world-1 line (short check)
TAG=${1:-bq}
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench $?
tail -1 gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['parity'], d['cpu_baseline']['value'], d['gpu_launches'])"
timeout 600 python bench.py --mode sharded --no-cpu-baseline > gpurun_out/bench_${TAG}_sh.log 2>&1; echo sh $?
tail -1 gpurun_out/bench_${TAG}_sh.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['parity'])"
