#!/bin/bash
# mixed-radix passes: parity + per-pass numbers vs the direct passes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed_radix.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/mixed_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mixed_tests.log
timeout 300 python tools/passbench.py 500x500x500,250x250x250,1000x1000,100x500x500 5 both > gpurun_out/passbench_mixed.jsonl 2> gpurun_out/passbench_mixed.err

tail -3 gpurun_out/mixed_tests.log
