# slab-decomposed path on the engine: world 1 vs engine/oracle, worlds 2/4 sharing the GPU
timeout 900 python -m pytest tests/test_gpu_slab.py -q -x > gpurun_out/gpu_slab.log 2>&1; tail -30 gpurun_out/gpu_slab.log
