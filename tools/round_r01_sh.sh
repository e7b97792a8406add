# data-dependent gate shortcuts (S == 0, spat_cur == 0, residual) + fused eps0/R2C: parity + bench A/B
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['lib_timings_ms'], d['e2e']['value'], d['roofline']['frac'])"
FFCZ_EPS0_FUSION=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_nofuse.log 2>&1; tail -1 gpurun_out/bench_nofuse.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no eps0 fusion', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_1024.log 2>&1; tail -1 gpurun_out/bench_c4_1024.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['lib_timings_ms'])"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_sh.csv $B > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_sh.csv > gpurun_out/launches_sh.txt; head -24 gpurun_out/launches_sh.txt
