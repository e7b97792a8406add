# 2-CTA cluster column pass: engine parity + per-pass micro-bench + frames / 1024^3 benches (A/B)
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_batch.py -q -x > gpurun_out/t_c2.log 2>&1; tail -3 gpurun_out/t_c2.log
timeout 300 python tools/passbench.py 1024x1024x1024,64x2048x2048 3 f64 > gpurun_out/pb_c2.log 2>&1; grep col_ gpurun_out/pb_c2.log
FFCZ_COL_C2=0 timeout 300 python tools/passbench.py 1024x1024x1024,64x2048x2048 3 f64 2>&1 | grep col_
timeout 900 python bench.py --config frames --frames 256 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c2_fr.log 2>&1; tail -1 gpurun_out/bench_c2_fr.log | cut -c 1-200
timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_c4.log 2>&1; tail -1 gpurun_out/bench_c2_c4.log | cut -c 1-200
