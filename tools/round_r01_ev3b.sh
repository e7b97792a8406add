# evidence pass 3 artifacts (ncu reps summarised on the box, then removed: gpurun_out <= 64 MiB)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c 1-150
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c 1-150
timeout 900 python bench.py --config combustion --n 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_1024.log 2>&1; tail -1 gpurun_out/bench_c4_1024.log | cut -c 1-150
timeout 900 python bench.py --config frames --frames 1024 --steps 3 --warmup 3 > gpurun_out/bench_frames1024.log 2>&1; tail -1 gpurun_out/bench_frames1024.log | cut -c 1-150
timeout 600 python tools/passbench.py 1024 5 > gpurun_out/passbench_1024.log 2>&1
timeout 600 python tools/passbench.py 512 10 > gpurun_out/passbench_512.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_ev3.csv $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'HookRepairVerifyS' -c 1 -o /tmp/prof_repair $B > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col_tma1' -c 1 -o /tmp/prof_outer python tools/passbench.py 512x512x512 1 f64 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_repair.ncu-rep > gpurun_out/ncu_repair.txt 2>&1
python tools/ncu_summary.py /tmp/prof_outer.ncu-rep > gpurun_out/ncu_outer.txt 2>&1
du -sh gpurun_out
