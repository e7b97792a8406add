#!/bin/bash
mkdir -p gpurun_out
FFCZ_GATE_ROW_FUSED=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_apply.py -x -q -m gpu > gpurun_out/grf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/grf_tests.log
for v in 0 1; do FFCZ_GATE_ROW_FUSED=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('fused=$v', d['value'], d['ms_per_step'], d['lib_timings_ms']['t_gate_ms'], d['escapes'], d['escape_rounds'] if 'escape_rounds' in d else '')"; done
tail -2 gpurun_out/grf_tests.log
