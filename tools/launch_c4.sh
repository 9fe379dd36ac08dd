B="python tools/blend_ab.py --config c4 --frames 4 --reps 1"
$B > gpurun_out/plain_l4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_l4.log 2>&1
B="python tools/blend_ab.py --frames 8 --reps 1"
$B > gpurun_out/plain_l3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_l3.log 2>&1
