timeout 900 python -m pytest tests/test_gpu_loop_rt.py tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_big.py tests/test_gpu_mixed.py -x -q -p no:cacheprovider > gpurun_out/el_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/el_pytest.log
for v in "" "FFCZ_LOOP_EPS_LATE=0"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$v', round(d['value'],3), round(d['ms_per_step'],1), d['lib_timings_ms']['t_loop_ms'], d['lib_timings_ms']['t_gate_ms'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernels'].items() if v['launches']})"
done
