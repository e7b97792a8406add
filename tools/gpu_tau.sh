timeout 900 python tools/tau_sweep.py 1024 1e-4,1e-5,1e-6,1e-7 > gpurun_out/tau_sweep.jsonl 2> gpurun_out/tau_sweep.err; echo "rc=$?"
