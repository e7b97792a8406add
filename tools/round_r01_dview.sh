#!/bin/bash
# decoder-view escape repair: full GPU suite, the rho-bound case that failed verify, the bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_suite.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite.log
timeout 300 python tools/debug_rho.py 256 512 > gpurun_out/debug_rho.log 2>&1
FFCZ_REPAIR_ORDER=reference timeout 300 python tools/debug_rho.py 512 >> gpurun_out/debug_rho.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_dview.log 2>&1
tail -3 gpurun_out/gpu_suite.log; cat gpurun_out/debug_rho.log; tail -1 gpurun_out/bench_dview.log | cut -c1-600
