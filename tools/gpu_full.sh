# round-end style evidence: full GPU suite, smoke, default bench line, the reference arm, and one
# ncu --set full capture of the dominant kernel class (plain outer-axis pass), summarised as text
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/full_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/full_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/full_ref.json 2> gpurun_out/full_ref.err; echo "ref rc=$?"
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:.*k_col_tma1<double, .int.1024, .int.16, .int.-1, ffcz_gpu::HookNone.*" -s 4 -c 1 --csv --page details python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/full_ncu_outer.csv 2>/dev/null; echo "ncu rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:.*(k_col_tma1_rt|k_row_c2r_r2c_sh).*" -s 4 -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-other-policy > gpurun_out/full_ncu_fused_dram.csv 2>/dev/null; echo "ncu2 rc=$?"
