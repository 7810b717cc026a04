#!/bin/bash
# Quick GPU iteration: build check, GPU tests (optionally filtered), short bench.
# usage: tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-}
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -2
if [ -n "$K" ]; then timeout 900 python -m pytest tests -q -m gpu -x -k "$K" > gpurun_out/tests_$TAG.log 2>&1; tail -15 gpurun_out/tests_$TAG.log
else timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/tests_$TAG.log 2>&1; tail -3 gpurun_out/tests_$TAG.log; fi
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo bench $?; tail -1 gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('it/s', d['value'], 'e2e', d['e2e']['value'], json.dumps(d['roofline']['per_family']), d['final_row'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l $?
