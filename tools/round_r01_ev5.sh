#!/bin/bash
# evidence pass 5: full suite (incl. slab decoder-view repair), smoke, frames line with launches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --config frames --frames 1024 --steps 3 --warmup 3 > gpurun_out/bench_frames1024.log 2>&1; tail -1 gpurun_out/bench_frames1024.log | cut -c 1-120
timeout 900 python bench.py --config slab --n 1024 --steps 3 --warmup 3 > gpurun_out/bench_slab1024.log 2>&1; tail -1 gpurun_out/bench_slab1024.log | cut -c 1-160
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c 1-160
