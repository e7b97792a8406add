#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/rowbudget.log
for b in 512 1024 2048; do
  FFCZ_TILE_BUDGET64_ROW=$b timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); k=d['kernels']
print($b, round(d['value'],2), round(d['ms_per_step'],3), {n:round(v['ms'],2) for n,v in k.items() if v['launches']})" >> gpurun_out/rowbudget.log
done
cat gpurun_out/rowbudget.log
