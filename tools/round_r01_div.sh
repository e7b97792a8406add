#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_suite.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_div.log 2>&1
tail -3 gpurun_out/gpu_suite.log
tail -1 gpurun_out/bench_div.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['lib_timings_ms']['t_gate_ms'], d['kernels'].get('elem_gate_quantize'), d['kernels'].get('elem_codes'))"
