#!/bin/bash
# ncu --set full (with source) of the C4 binning kernels: k_row_scatter,
# k_row_items, the row-partition onesweep and k_bin_offsets (one frame each)
mkdir -p gpurun_out/r02bin
python -m paper_2503_16422_b200.build > gpurun_out/r02bin/build.log 2>&1
A="python tools/blend_ab.py --config c4 --frames 2 --reps 1"
$A > gpurun_out/r02bin/plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_row_scatter|k_row_items|k_bin_offsets|k_bin_count|k_row_count" -s 15 -c 5 \
  -o gpurun_out/r02bin/prof_bin $A > gpurun_out/r02bin/ncu.log 2>&1
echo "bin rc=$?"
