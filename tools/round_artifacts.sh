#!/bin/bash
# (round 1; flags as of round 1 -- bench.py now defaults to front-end graphs, --no-graphs for stream launches)
# Round artifacts on the GPU box: bench lines (c3 default, c3 VQ, c2, c4 masked
# and unmasked), STV probe, sweeps, then the launch list and ncu captures.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --vq 4096 --no-cpu-baseline > gpurun_out/bench_c3_vq.json 2>&1
python bench.py --literal-masks --no-cpu-baseline > gpurun_out/bench_c3_literal.json 2>&1
python bench.py --config c2 --no-cpu-baseline --streams 12 > gpurun_out/bench_c2.json 2>&1
python bench.py --config c4 --no-cpu-baseline --steps 4 > gpurun_out/bench_c4_masked.json 2>&1
python bench.py --config c4 --unmasked --no-cpu-baseline --steps 4 > gpurun_out/bench_c4_unmasked.json 2>&1
python tools/stv_probe.py > gpurun_out/stv_probe.json 2>&1
timeout 900 python tools/sweeps.py > gpurun_out/sweeps.json 2> gpurun_out/sweeps.err
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
