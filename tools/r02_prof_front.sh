#!/bin/bash
# Per-kernel duration / instructions / occupancy of the front end at C3 and C4
# (serialised ncu launch list; compare shares, not absolutes)
mkdir -p gpurun_out
python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1
for c in c3 c4; do
  A="python tools/blend_ab.py --config $c --frames 6 --reps 1"
  $A > gpurun_out/plain_front_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -s 200 -c 120 --csv --log-file gpurun_out/front_$c.csv $A > gpurun_out/ncu_front_$c.log 2>&1
  echo "$c rc=$?"
done
