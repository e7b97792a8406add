#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/m1000.jsonl
for kb in 96 144 200; do
  echo "{\"pipe_kb\": $kb}" >> gpurun_out/m1000.jsonl
  FFCZ_MIXED_PIPE_KB=$kb timeout 300 python tools/passbench.py 1000x1000x1000 3 f64 2>/dev/null | grep col >> gpurun_out/m1000.jsonl
done
for kb in 64 128; do
  echo "{\"row_kb\": $kb}" >> gpurun_out/m1000.jsonl
  FFCZ_MIXED_SMEM=$kb timeout 300 python tools/passbench.py 1000x1000x1000 3 f64 2>/dev/null | grep row >> gpurun_out/m1000.jsonl
done
cat gpurun_out/m1000.jsonl
