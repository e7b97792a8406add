# mixed policy: tests + timing vs fp64 on the config-4 recipe (512^3, 1024^3)
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_parity.py -q -x > gpurun_out/gpu_mixed.log 2>&1; tail -15 gpurun_out/gpu_mixed.log
for n in 512 1024; do for pol in fp64 mixed; do
timeout 900 python bench.py --config combustion --n $n --policy $pol --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_${n}_$pol.log 2>&1; echo "$n $pol"; tail -1 gpurun_out/bench_c4_${n}_$pol.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['iterations'], d.get('iterations_fp32'), d['lib_timings_ms'])"
done; done
timeout 300 python tools/passbench.py 1024 3 f32 2>&1 | grep -v 2048
