#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/frames_budget.log
for gb in 30 60 100 130; do
  FFCZ_FRAMES_BUDGET_GB=$gb timeout 600 python bench.py --config frames --frames 1024 --steps 2 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "
import sys,json
try:
    d=json.loads(sys.stdin.read()); print($gb, round(d['value'],2), round(d['ms_per_step'],1), round(d['loop_ms_per_step'],1), d['clocks']['reasons'])
except Exception as e: print($gb, 'failed', e)" >> gpurun_out/frames_budget.log
done
cat gpurun_out/frames_budget.log
