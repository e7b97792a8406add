# A/B of runtime switches on the default bench workload (device value only), one line per setting:
#   bash tools/gpu_ab.sh "" "FFCZ_X=1" "FFCZ_Y=0 FFCZ_Z=1" ...
for v in "$@"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('[$v]', round(d['value'],3), round(d['ms_per_step'],1), round(d['lib_timings_ms']['t_loop_ms'],1), round(d['lib_timings_ms']['t_gate_ms'],1), {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernels'].items() if v['launches']})"
done
