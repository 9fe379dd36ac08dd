#!/bin/bash
# Round-2 profile on the GPU box (one GPU): the launch list of a short bench run
# with per-launch duration, warp instructions and DRAM bytes, and one ncu
# --set full capture (with source) of the timed blend.  Each ncu command first
# runs plain and must exit 0.
mkdir -p gpurun_out/r02prof
python -m paper_2503_16422_b200.build --force > gpurun_out/r02prof/build.log 2>&1
B="python bench.py --steps 1 --warmup 3 --frames-per-step 20 --no-e2e --no-cpu-baseline --no-stage-events"
$B > gpurun_out/r02prof/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02prof/launches.csv $B > gpurun_out/r02prof/ncu_launches.log 2>&1
echo "launches rc=$?"
A="python tools/blend_ab.py --frames 8 --reps 1"
$A > gpurun_out/r02prof/plain_ab.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_blend_wi" -s 8 -c 2 -o gpurun_out/r02prof/prof_blend -f $A > gpurun_out/r02prof/ncu_blend.log 2>&1
echo "blend rc=$?"
ls -la gpurun_out/r02prof
