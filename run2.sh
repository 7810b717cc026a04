set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' 2>&1 | tail -3
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -30
timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -3
timeout 300 python bench.py --config 2 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -3
