timeout 900 python -m pytest tests/test_gpu_loop_rt.py tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_repair_order.py tests/test_gpu_big.py -x -q -p no:cacheprovider > gpurun_out/rt6_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/rt6_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/rt6_bench.json 2> gpurun_out/rt6_bench.err; echo "bench rc=$?"
