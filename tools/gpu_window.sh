#!/bin/bash
# the bench over different iteration windows (early iterations: clumped cells)
for w in 3 5 20 60 120; do
  timeout 600 python bench.py --steps 20 --warmup $w --no-cpu-baseline > gpurun_out/win_$w.log 2>&1
  tail -1 gpurun_out/win_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=$w', round(d['value'],1), d['roofline']['stages_us'], d['critical_path_us'])"
done
