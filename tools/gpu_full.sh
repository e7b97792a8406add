# round-end style evidence: full GPU suite, smoke, default bench line
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/full_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/full_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "bench rc=$?"
