timeout 300 python tools/passbench.py 512 10 > gpurun_out/passbench_default.log 2>&1
FFCZ_CUDA_LIB=$PWD/paper_2601_01596_b200/libffcz_cuda_e8.so timeout 300 python tools/passbench.py 512 10 > gpurun_out/passbench_e8.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -c 1500 gpurun_out/bench.log
