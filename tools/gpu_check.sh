set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s5_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/s5_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --config nyx > gpurun_out/s5_bench_nyx.json 2> gpurun_out/s5_bench_nyx.err; echo "nyx rc=$?"
