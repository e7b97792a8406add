# repair-round C2R with bulk-copy input prefetch: parity + bench + launch list
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['lib_timings_ms'], d['e2e']['value'], d['roofline']['frac'])"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_pf.csv $B > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_pf.csv | head -8
timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_1024.log 2>&1; tail -1 gpurun_out/bench_c4_1024.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['lib_timings_ms'])"
