A="python tools/blend_ab.py --config c4 --frames 6 --reps 1"
$A > gpurun_out/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_cull|k_slice" -s 12 -c 2 -o gpurun_out/prof_c4 $A > gpurun_out/ncu_c4.log 2>&1
cat gpurun_out/plain_c4.log
