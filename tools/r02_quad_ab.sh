#!/bin/bash
mkdir -p gpurun_out
python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
for r in 1 2; do for v in wi q12 q10 q8 q12u4; do echo -n "$v "; AB_LIB=tools/variants/libfdgs_$v.so python tools/blend_ab.py --frames 24 --reps 5; done; done
python tools/pipe_ab.py --rounds 4 --steps 5 native:4#wi native:4#q12 native:4#q10 native:4#q8
