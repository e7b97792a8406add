# one ncu --set full capture of the loop's fused kernels (round trip + K1) at 1024^3 config 4
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_col_tma1_rt|k_row_c2r_r2c_sh" -s 6 -c 2 -o gpurun_out/loop_ncu python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/loop_ncu.log 2>&1; echo "ncu rc=$?"
