# A/B of the TMA-staged column pass against the register-direct one, then parity + bench
timeout 300 python tools/passbench.py 512 10 > gpurun_out/pb_tma.log 2>&1
FFCZ_COL_TMA=0 timeout 300 python tools/passbench.py 512 10 > gpurun_out/pb_direct.log 2>&1
for b in 4 16; do FFCZ_COL_TMA_B=$b timeout 300 python tools/passbench.py 512 10 > gpurun_out/pb_tma_b$b.log 2>&1; done
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -c 1500 gpurun_out/bench.log
