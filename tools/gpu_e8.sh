timeout 600 python -m pytest tests/test_gpu_mixed.py -x -q -p no:cacheprovider > gpurun_out/e8_mixed.log 2>&1; echo "mixed rc=$?"; tail -1 gpurun_out/e8_mixed.log
FFCZ_TMA1_E8=1 timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity.py tests/test_gpu_loop_rt.py -x -q -p no:cacheprovider > gpurun_out/e8_pytest.log 2>&1; echo "e8 pytest rc=$?"; tail -1 gpurun_out/e8_pytest.log
for v in "" "FFCZ_TMA1_E8=1"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$v', round(d['value'],3), round(d['ms_per_step'],1), d['lib_timings_ms']['t_loop_ms'], d['lib_timings_ms']['t_gate_ms'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernels'].items() if v['launches']})"
done
