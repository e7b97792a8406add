# why is the 1024^3 outer-axis pass ~2x slower under CUDA events than under ncu?
nvidia-smi dmon -s pucv -d 1 > gpurun_out/dmon_1024.log 2>&1 &
DM=$!
for r in 1 3 20; do echo "reps=$r"; timeout 300 python tools/passbench.py 1024x1024x1024 $r f64 2>&1 | grep -E "col_|row_"; done
sleep 2; kill $DM
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_col' --csv --log-file gpurun_out/launches_pb1024.csv python tools/passbench.py 1024x1024x1024 3 f64 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_pb1024.csv
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:'k_col' --csv --log-file gpurun_out/launches_pb1024_nc.csv python tools/passbench.py 1024x1024x1024 3 f64 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_pb1024_nc.csv
