#!/bin/bash
mkdir -p gpurun_out
for k in k_col_mixed_pipe k_row_r2c_mixed; do
timeout 600 ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -f -o /tmp/ncu_$k python tools/passbench.py 500x500x500 1 f64 > /dev/null 2>&1
ncu -i /tmp/ncu_$k.ncu-rep --page details --csv > gpurun_out/ncu2_${k}_details.csv 2>&1
done
