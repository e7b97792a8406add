#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/mixed_sweep.jsonl
timeout 600 python -m pytest tests/test_gpu_mixed_radix.py -x -q -m gpu > gpurun_out/mixed_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mixed_tests.log
for kb in 48 72 96 144; do
  echo "{\"pipe_kb\": $kb}" >> gpurun_out/mixed_sweep.jsonl
  FFCZ_MIXED_PIPE_KB=$kb timeout 200 python tools/passbench.py 500x500x500,1000x1000,250x250x250 5 both >> gpurun_out/mixed_sweep.jsonl 2>> gpurun_out/mixed_sweep.err
done
tail -2 gpurun_out/mixed_tests.log
