# batched frames: GPU parity of correct_batch + config-3 bench (1024 frames of 2048^2 at 1 GPU)
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py --config frames --frames 256 --steps 3 --warmup 3 > gpurun_out/bench_frames256.log 2>&1; tail -c 2500 gpurun_out/bench_frames256.log
for L in 4 16; do timeout 900 python bench.py --config frames --frames 256 --lanes $L --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_frames256_l$L.log 2>&1; tail -1 gpurun_out/bench_frames256_l$L.log | cut -c 1-300; done
