#!/bin/bash
# Build libfdgs.so variants for A/B timing: tools/ab_build.sh NAME "-DFLAG=..." ...
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/variants
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o tools/variants/libfdgs_${name}.so paper_2503_16422_b200/csrc/{render,aux,stv,api,pipeline}.cu
