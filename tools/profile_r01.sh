set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ffcz_gpu --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_row_r2c -s 3 -c 1 -o gpurun_out/prof_row_r2c $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_col -s 6 -c 1 -o gpurun_out/prof_col $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_row_c2r_r2c -s 1 -c 1 -o gpurun_out/prof_row_fused $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_row_c2r -s 3 -c 1 -o gpurun_out/prof_row_c2r $B > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_shim.py -q > gpurun_out/shim.log 2>&1
ls -la gpurun_out
