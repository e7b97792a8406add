# device Huffman encoder: parity vs the reference payload + archive timing at 512^3
timeout 900 python -m pytest tests/test_gpu_encode.py -q -x > gpurun_out/gpu_encode.log 2>&1; tail -15 gpurun_out/gpu_encode.log
timeout 1200 python tools/archive_time.py 512 > gpurun_out/archive_time.log 2>&1; tail -6 gpurun_out/archive_time.log
