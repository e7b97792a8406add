# frames: where does the time go (sum of kernel durations vs wall)
B="python bench.py --config frames --frames 128 --steps 1 --warmup 1 --no-e2e"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_frames.csv $B > gpurun_out/ncu_frames.log 2>&1
python tools/launches.py gpurun_out/launches_frames.csv 5 > gpurun_out/launches_frames.txt; head -40 gpurun_out/launches_frames.txt
timeout 600 python bench.py --config frames --frames 128 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_f128.log 2>&1; tail -1 gpurun_out/bench_f128.log | cut -c 1-250
