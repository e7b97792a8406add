B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1
tail -3 gpurun_out/ncu_launch_stdout.log
