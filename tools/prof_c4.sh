A="python tools/blend_ab.py --config c4 --frames 6 --reps 1"
$A > gpurun_out/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_bin_scan|k_row_items|k_row_scatter|k_row_count|k_onesweep" -s 30 -c 12 -o gpurun_out/prof_c4 $A > gpurun_out/ncu_c4.log 2>&1
cat gpurun_out/plain_c4.log
