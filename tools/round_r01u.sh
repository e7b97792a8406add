# memcheck the correct() paths the encode-archive tests exercise (twiddle-table corruption hunt)
timeout 1500 compute-sanitizer --tool memcheck --print-limit 30 python -m pytest tests/test_gpu_encode.py -q -x -k "archive" > gpurun_out/t_memcheck2.log 2>&1; grep -E "ERROR SUMMARY|Invalid|at 0x|by thread|Address|passed|failed" gpurun_out/t_memcheck2.log | head -40
for k in accept_05 config1_c1.0 config3_frame256 odd_12x10x9 m8_32cube config2_rho32 config4_comb32; do
timeout 300 python -m pytest "tests/test_gpu_encode.py::test_device_encoded_archive[$k]" tests/test_gpu_engine.py -q -x > gpurun_out/t_k.log 2>&1; echo "$k: $(tail -1 gpurun_out/t_k.log)"; done
