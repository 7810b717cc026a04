python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_loop.py -q -x -k bit_identical 2>&1 | tail -15
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['final_row'])"; done
