# outer-axis 256-B tiles (k_col_tma1, E=16 at L=512): pass micro-bench + parity + headline bench + archive timing
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python tools/passbench.py 512x512x512,1024x512x512,512x1024x1024 5 f64 > gpurun_out/pb_new.log 2>&1; grep col_ gpurun_out/pb_new.log
FFCZ_COL_TMA1=0 timeout 300 python tools/passbench.py 512x512x512 5 f64 2>&1 | grep col_
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c 1-500
timeout 1500 python tools/archive_time.py 512 > gpurun_out/archive_time.log 2>&1; tail -6 gpurun_out/archive_time.log
