# A/B of runtime switches on the default bench workload (device value only)
for v in "" "FFCZ_GATE_ROW_FUSED=1" "FFCZ_LOOP_K1=0" "FFCZ_LOOP_RT=0"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$v', round(d['value'],3), round(d['ms_per_step'],1), d['lib_timings_ms']['t_loop_ms'], d['lib_timings_ms']['t_gate_ms'])"
done
