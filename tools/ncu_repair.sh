#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_metrics.py -q -m gpu > gpurun_out/metrics_tests.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'HookRepairVerifyS' -c 1 -f -o /tmp/prof_repair $B > gpurun_out/ncu_repair.log 2>&1
ncu -i /tmp/prof_repair.ncu-rep --page details --csv > gpurun_out/prof_repair_details.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'k_gate_freq' -c 1 -f -o /tmp/prof_gate $B > gpurun_out/ncu_gate.log 2>&1
ncu -i /tmp/prof_gate.ncu-rep --page details --csv > gpurun_out/prof_gate_details.csv 2>&1
tail -1 gpurun_out/metrics_tests.log
