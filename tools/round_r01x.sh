# unrolled gate kernels: parity + bench; escape composition at 512^3
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['lib_timings_ms'], d['e2e']['value'])"
timeout 600 python tools/escape_split.py 512 > gpurun_out/escape_split.log 2>&1; tail -2 gpurun_out/escape_split.log
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_r01x.csv $B > /dev/null 2>&1
