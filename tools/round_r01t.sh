# isolate the 256^3 FP64 R2C failure: engine tests alone, then after the encoder tests; memcheck the encoder
timeout 600 python -m pytest tests/test_gpu_engine.py -q -x > gpurun_out/t_engine.log 2>&1; tail -2 gpurun_out/t_engine.log
timeout 600 python -m pytest tests/test_gpu_encode.py tests/test_gpu_engine.py -q -x > gpurun_out/t_enc_engine.log 2>&1; tail -2 gpurun_out/t_enc_engine.log
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_engine.py -q -x > gpurun_out/t_batch_engine.log 2>&1; tail -2 gpurun_out/t_batch_engine.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_encode.py -q -x -k "payload" > gpurun_out/t_memcheck.log 2>&1; grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/t_memcheck.log | head -20
