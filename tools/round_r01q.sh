# slab path: GPU tests + throughput at world 1 (config-4 recipe)
timeout 900 python -m pytest tests/test_gpu_slab.py -q -x > gpurun_out/gpu_slab.log 2>&1; tail -3 gpurun_out/gpu_slab.log
timeout 900 python bench.py --config slab --n 512 --steps 3 --warmup 3 > gpurun_out/bench_slab512.log 2>&1; tail -1 gpurun_out/bench_slab512.log | cut -c 1-400
timeout 1200 python bench.py --config slab --n 1024 --steps 3 --warmup 3 > gpurun_out/bench_slab1024.log 2>&1; tail -1 gpurun_out/bench_slab1024.log | cut -c 1-400
