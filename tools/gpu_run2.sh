bash tools/gpu_ab.sh "" "FFCZ_EPS0_FUSION=1" "FFCZ_GATE_ROW_FUSED=1"
SECS="--section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section LaunchStats --section Occupancy --section SchedulerStats"
FFCZ_GATE_ROW_FUSED=1 timeout 900 ncu $SECS --clock-control none --kernel-name-base demangled -k "regex:.*RepairVerifyS.*" -s 1 -c 1 --csv --page details python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/gate_row_fused.csv 2>/dev/null; echo "ncu1 rc=$?"
timeout 900 ncu $SECS --clock-control none --kernel-name-base demangled -k "regex:.*RepairVerifyS.*" -s 1 -c 1 --csv --page details python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/gate_row_split.csv 2>/dev/null; echo "ncu2 rc=$?"
ls -la gpurun_out/
