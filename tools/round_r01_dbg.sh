timeout 600 python -m pytest tests/test_gpu_apply.py -v -x 2>&1 | tail -15
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_apply.py -q -x -k "engine_archive" > gpurun_out/memcheck_pf.log 2>&1; grep -E "ERROR SUMMARY|Invalid|Address|at 0x|by thread|passed|failed|Error" gpurun_out/memcheck_pf.log | head -30
