# Round-1 evidence pass: GPU tests, smoke, bench, per-pass micro-bench, ncu launch list + one full capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log
timeout 300 python tools/passbench.py 512 10 > gpurun_out/passbench.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch_stdout.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_col' -s 20 -c 1 -o gpurun_out/prof_col $B > gpurun_out/ncu_full_stdout.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:'k_row_c2r_r2c' -s 2 -c 1 -o gpurun_out/prof_row_fused $B >> gpurun_out/ncu_full_stdout.log 2>&1
ls -la gpurun_out
