# F rebuild (clip byte map + one forward at the gate) vs per-pass F read-modify-write
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
FFCZ_F_REBUILD=0 timeout 900 python -m pytest tests -q -m gpu -x -k "parity" > gpurun_out/gpu_tests_norebuild.log 2>&1; tail -1 gpurun_out/gpu_tests_norebuild.log
for fr in 1 0; do
FFCZ_F_REBUILD=$fr timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_1024_fr$fr.log 2>&1; echo "rebuild=$fr"; tail -1 gpurun_out/bench_c4_1024_fr$fr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['iterations'], d['lib_timings_ms'])"
done
timeout 600 python bench.py --config combustion --n 512 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_512.log 2>&1; tail -1 gpurun_out/bench_c4_512.log | cut -c 1-600
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c 1-600
