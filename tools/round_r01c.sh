for b in 2048 1024 8192; do FFCZ_TILE_BUDGET64=$b timeout 300 python tools/passbench.py 512 10 2>&1 | grep '"f64"' | grep -v 2048, > gpurun_out/passbench_b$b.log; done
FFCZ_DEBUG_TIMING=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_dbg.log 2>&1
tail -c 600 gpurun_out/bench_dbg.log
