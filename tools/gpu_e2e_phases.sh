# phase timings of correct() + the device archive at 1024^3 config 4 through the e2e path
FFCZ_DEBUG_TIMING=1 timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-policy > gpurun_out/e2e_phases.json 2> gpurun_out/e2e_phases.err; echo "rc=$?"
