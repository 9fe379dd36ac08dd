#!/bin/bash
# Round-2 probe on the GPU box: build, GPU tests, default bench, isolated stage
# times, and one ncu --set full capture (with source counters) of the timed blend.
mkdir -p gpurun_out
python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1 || exit 1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/blend_ab.py --frames 24 --reps 5 > gpurun_out/blend_ab.json 2>&1; echo "ab rc=$?"; cat gpurun_out/blend_ab.json
A="python tools/blend_ab.py --frames 8 --reps 1"
$A > gpurun_out/plain_ab.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_blend_wi" -s 8 -c 2 -o gpurun_out/prof_blend -f $A > gpurun_out/ncu_blend.log 2>&1; echo "ncu rc=$?"
