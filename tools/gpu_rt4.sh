timeout 900 python -m pytest tests/test_gpu_loop_rt.py tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_repair_order.py tests/test_gpu_mixed.py -x -q -p no:cacheprovider > gpurun_out/rt4_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/rt4_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/rt4_bench.json 2> gpurun_out/rt4_bench.err; echo "bench rc=$?"
