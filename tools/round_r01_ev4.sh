#!/bin/bash
# evidence pass 4 (end of session): suite, smoke, bench lines, launch list, one full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c 1-150
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c 1-150
timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_1024.log 2>&1; tail -1 gpurun_out/bench_c4_1024.log | cut -c 1-150
timeout 900 python bench.py --config frames --frames 1024 --steps 3 --warmup 3 > gpurun_out/bench_frames1024.log 2>&1; tail -1 gpurun_out/bench_frames1024.log | cut -c 1-150
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_ev4.csv $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'HookRepairVerifyS' -c 1 -f -o /tmp/prof_repair $B > /dev/null 2>&1
ncu -i /tmp/prof_repair.ncu-rep --page details --csv > gpurun_out/prof_repair_details.csv 2>&1
ncu -i /tmp/prof_repair.ncu-rep --page raw --csv > gpurun_out/prof_repair_raw.csv 2>&1
ls -la gpurun_out/ | tail -20
