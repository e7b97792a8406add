# device decoder tests + clean ncu --set full captures of the pass kernels (passbench, no gating)
timeout 900 python -m pytest tests/test_gpu_apply.py -q -x > gpurun_out/gpu_apply.log 2>&1; tail -15 gpurun_out/gpu_apply.log
P="python tools/passbench.py 512x512x512 1 f64"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col_tma1' -c 1 -o gpurun_out/prof_outer $P > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col_tma<' -c 1 -o gpurun_out/prof_mid $P > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_row_r2c' -c 1 -o gpurun_out/prof_r2c $P > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'HookRepairVerifyS' -c 1 -o gpurun_out/prof_repair $B > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
