# launch list of the default bench command (kernel durations, cold-cache, serialised) + RT E8 A/B
for v in "FFCZ_RT_E8=1"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$v', round(d['value'],3), round(d['ms_per_step'],1), d['lib_timings_ms']['t_loop_ms'], d['lib_timings_ms']['t_gate_ms'], {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernels'].items() if v['launches']})"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r02b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/launches_r02b.log 2>&1; echo "ncu rc=$?"
