#!/bin/bash
# Round profile on the GPU box: launch list of the bench command and one full
# ncu capture of the timed blend.  Each ncu command line first runs plain (exit 0).
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --frames-per-step 20 --no-e2e --no-cpu-baseline --no-stage-events"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
A="python tools/blend_ab.py --frames 8 --reps 1"
$A > gpurun_out/plain_ab.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_blend_wi|k_slice|k_row_scatter|k_row_items" -s 24 -c 4 -o gpurun_out/prof_full $A > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
