timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_batch.py tests/test_gpu_big.py tests/test_gpu_loop_rt.py tests/test_gpu_mixed.py tests/test_gpu_apply.py tests/test_gpu_repair_order.py -x -q -p no:cacheprovider > gpurun_out/r4_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r4_pytest.log
bash tools/gpu_ab.sh ""
