# full GPU suite after the stream-ordering fix; headline bench line; ncu launch list + full captures
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c 1-300
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_r01v.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col_tma1' -s 4 -c 1 -o gpurun_out/prof_outer $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col_tma<double, 512, 8, 1, HookNone' -s 2 -c 1 -o gpurun_out/prof_mid $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_row_c2r_sh<double, 256, 16, HookRepairVerifyS' -s 1 -c 1 -o gpurun_out/prof_repair $B > /dev/null 2>&1
ls gpurun_out
