# batched-frame fused loop: parity vs per-frame correct(), frames bench fused vs lanes
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/gpu_batch.log 2>&1; tail -15 gpurun_out/gpu_batch.log
timeout 900 python bench.py --config frames --frames 256 --steps 3 --warmup 3 > gpurun_out/bench_frames256.log 2>&1; tail -1 gpurun_out/bench_frames256.log | cut -c 1-400
FFCZ_FRAMES_FUSED=0 timeout 900 python bench.py --config frames --frames 256 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_frames256_lanes.log 2>&1; tail -1 gpurun_out/bench_frames256_lanes.log | cut -c 1-300
cat gpurun_out/round_r01y_note 2>/dev/null
