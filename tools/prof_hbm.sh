# ncu DRAM evidence for the HBM-side kernels (cull, slice, emits, sorts) at C3 and C4
for c in c3 c4; do
A="python tools/blend_ab.py --config $c --frames 4 --reps 1"
$A > gpurun_out/plain_hbm_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_cull|k_slice|k_vis_emit|k_onesweep|k_sort_hist|k_row_items|k_row_scatter|k_blend_wi" -s 60 -c 16 --csv --log-file gpurun_out/hbm_$c.csv $A > gpurun_out/ncu_hbm_$c.log 2>&1
done
