# batched per-frame gate: parity (batch tests compare with per-frame correct()) + frames bench
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/gpu_batch.log 2>&1; tail -30 gpurun_out/gpu_batch.log
timeout 900 python bench.py --config frames --frames 256 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_bg256.log 2>&1; tail -1 gpurun_out/bench_bg256.log | cut -c 1-300
timeout 900 python bench.py --config frames --frames 1024 --steps 3 --warmup 3 > gpurun_out/bench_bg1024.log 2>&1; tail -1 gpurun_out/bench_bg1024.log | cut -c 1-300
