timeout 1200 python -m pytest tests/test_gpu_slab.py -x -q -p no:cacheprovider > gpurun_out/slab_pytest.log 2>&1; echo "slab pytest rc=$?"; tail -1 gpurun_out/slab_pytest.log
for v in "" "FFCZ_SLAB_FUSED_ROW=0"; do
  env $v timeout 900 python bench.py --config slab --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/slab_ab.json 2>gpurun_out/slab_ab.err
  python -c "
import json;d=json.loads(open('gpurun_out/slab_ab.json').read().strip().splitlines()[-1]); print('[$v]', d['value'], d['ms_per_step'])" || tail -3 gpurun_out/slab_ab.err
done
