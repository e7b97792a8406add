timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/gpu_batch.log 2>&1; tail -30 gpurun_out/gpu_batch.log | grep -E "passed|failed|Error|assert" | head
FFCZ_FRAMES_BATCHED_GATE=0 timeout 900 python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -1
