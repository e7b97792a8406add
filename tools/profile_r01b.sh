B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1
# first-axis pass with the per-component check (K3a), middle-axis plain pass, row C2R with the repair hook
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col<double, 512, 8, -1, HookFReduce' -s 1 -c 1 -o gpurun_out/prof_k3a $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col<double, 512, 8, -1, HookNone' -s 1 -c 1 -o gpurun_out/prof_colmid $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_row_r2c_sh' -s 2 -c 1 -o gpurun_out/prof_r2c_sh $B > /dev/null 2>&1
ls gpurun_out
