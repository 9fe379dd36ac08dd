A="python tools/blend_ab.py --frames 6 --reps 1"
$A > gpurun_out/plain_front.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_cull|k_slice|k_bin_scan|k_row_items|k_row_scatter|k_row_count|k_tile_scan|k_sort_hist|k_onesweep" -s 40 -c 11 -o gpurun_out/prof_front $A > gpurun_out/ncu_front.log 2>&1
tail -3 gpurun_out/ncu_front.log
