#!/bin/bash
# ncu DRAM evidence for the HBM-side kernels on the bench's path (compacted
# working sets) at C3 and C4: per-launch duration, DRAM bytes, achieved GB/s
# (cold cache, serialised).  tools/hbm_summary.py summarises the csv.
mkdir -p gpurun_out/r02hbm
python -m paper_2503_16422_b200.build > gpurun_out/r02hbm/build.log 2>&1
for c in c3 c4; do
  B="python bench.py --config $c --steps 2 --warmup 3 --frames-per-step 8 --no-e2e --no-cpu-baseline --no-stage-events"
  $B > gpurun_out/r02hbm/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_cull|k_slice|k_vis_emit|k_onesweep|k_sort_hist|k_bin_count|k_row_items|k_row_scatter|k_blend_wi|k_scene_gather|k_mask_compact" -s 400 -c 120 --csv --log-file gpurun_out/r02hbm/hbm_$c.csv $B > gpurun_out/r02hbm/ncu_$c.log 2>&1
  echo "$c rc=$?"
  python tools/hbm_summary.py gpurun_out/r02hbm/hbm_$c.csv > gpurun_out/r02hbm/summary_$c.txt 2>&1
done
