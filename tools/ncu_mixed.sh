#!/bin/bash
# ncu --set full of the mixed-radix passes at 500^3 FP64; reports stay in /tmp, summaries come back
mkdir -p gpurun_out
for k in k_col_mixed k_row_r2c_mixed; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o /tmp/ncu_$k python tools/passbench.py 500x500x500 1 f64 > gpurun_out/ncu_$k.log 2>&1
ncu -i /tmp/ncu_$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>&1
ncu -i /tmp/ncu_$k.ncu-rep --page details --csv > gpurun_out/ncu_${k}_details.csv 2>&1
ncu -i /tmp/ncu_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${k}_sass.csv 2>&1
done
du -sh gpurun_out/*
