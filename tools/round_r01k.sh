# A/B: single-landing first-axis pass (k_col_tma1) and middle-axis completion of the forward transform
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python tools/passbench.py 1024 5 > gpurun_out/pb1024_new.log 2>&1; grep -v 2048 gpurun_out/pb1024_new.log
FFCZ_COL_TMA1=0 timeout 300 python tools/passbench.py 1024 5 > gpurun_out/pb1024_old.log 2>&1; grep axis_first gpurun_out/pb1024_old.log
timeout 300 python tools/passbench.py 512 10 > gpurun_out/pb512_new.log 2>&1; grep -v 2048 gpurun_out/pb512_new.log
for za in 1 0; do
FFCZ_COMPLETE_AXIS=$za timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench512_za$za.log 2>&1; echo "za=$za"; tail -1 gpurun_out/bench512_za$za.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['lib_timings_ms'], d['e2e']['value'], json.dumps(d['kernels']))"
FFCZ_COMPLETE_AXIS=$za timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_1024_za$za.log 2>&1; tail -1 gpurun_out/bench_c4_1024_za$za.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['iterations'], d['lib_timings_ms'], json.dumps(d['kernels']))"
done
