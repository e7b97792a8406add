# frames: double-buffered groups with background per-frame gates
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/gpu_batch.log 2>&1; tail -2 gpurun_out/gpu_batch.log
timeout 900 python bench.py --config frames --frames 256 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_fo256.log 2>&1; echo "256: $(tail -1 gpurun_out/bench_fo256.log | cut -c 1-200)"
timeout 1500 python bench.py --config frames --frames 1024 --steps 3 --warmup 3 > gpurun_out/bench_fo1024.log 2>&1; tail -1 gpurun_out/bench_fo1024.log | cut -c 1-300
