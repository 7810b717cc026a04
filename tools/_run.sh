python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
timeout 600 python tools/e2e_probe.py 20 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --precision fp32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fp32 it/s', d['value'], json.dumps(d['roofline']['per_family']), d['final_row'])"
