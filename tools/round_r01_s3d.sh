#!/bin/bash
# non-power-of-two end to end (S3D-like 500^3 on the config-4 recipe) + full GPU suite
mkdir -p gpurun_out
timeout 900 python bench.py --config combustion --n 500 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_500.log 2>&1
timeout 900 python bench.py --config combustion --n 512 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_512.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_suite.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite.log
tail -1 gpurun_out/bench_c4_500.log; tail -1 gpurun_out/bench_c4_512.log; tail -3 gpurun_out/gpu_suite.log
