# frames: lanes for the per-frame gate phase; the full 1024-frame workload
for L in 8 16 32; do timeout 900 python bench.py --config frames --frames 256 --lanes $L --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_fr_l$L.log 2>&1; echo "lanes $L: $(tail -1 gpurun_out/bench_fr_l$L.log | cut -c 1-160)"; done
timeout 1500 python bench.py --config frames --frames 1024 --lanes 16 --steps 3 --warmup 3 > gpurun_out/bench_fr1024.log 2>&1; tail -1 gpurun_out/bench_fr1024.log | cut -c 1-400
