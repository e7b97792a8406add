timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/gpu_batch.log 2>&1; tail -15 gpurun_out/gpu_batch.log
