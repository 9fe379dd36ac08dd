#!/bin/bash
mkdir -p gpurun_out
python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1
python tools/blend_ab.py --frames 24 --reps 5
python tools/pipe_ab.py --rounds 4 --steps 5 native:4 native:4#sleep100 native:4#sleep400 native:4#sleep1500
python tools/pipe_ab.py --config c4 --rounds 3 --steps 3 native:4 native:4#sleep100 native:4#sleep400 native:4#sleep1500
A="python tools/blend_ab.py --config c4 --frames 2 --reps 1"
$A > gpurun_out/plain_sort.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_onesweep" -s 12 -c 2 -o gpurun_out/prof_sort -f $A > gpurun_out/ncu_sort.log 2>&1; echo ncu rc=$?
