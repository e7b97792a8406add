bash tools/gpu_ab.sh "" "FFCZ_TMA1_HALF=1"
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:.*k_col_tma1<double, .int.1024, .int.16, .int.-1, ffcz_gpu::HookNone.*" -s 4 -c 1 --csv --page details python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/full_ncu_outer.csv 2>/dev/null; echo "ncu rc=$?"
