# north-star size: config-4 recipe at 512^3 and 1024^3 on one B200 + per-pass micro-bench at 1024^3
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
free -g > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
timeout 600 python bench.py --config combustion --n 512 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_512.log 2>&1; tail -c 1500 gpurun_out/bench_c4_512.log
timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_1024.log 2>&1; tail -c 3000 gpurun_out/bench_c4_1024.log

