# bench the default build and an FP64 E<=8 variant, then the GPU test suite
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/bench_default.log 2>&1
FFCZ_CUDA_LIB=$PWD/paper_2601_01596_b200/libffcz_cuda_e8.so timeout 300 $B > gpurun_out/bench_e8.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
