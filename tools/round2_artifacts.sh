#!/bin/bash
# Round-2 bench lines on the GPU box (profiles/r02_*): every BASELINE config,
# cpu_baseline with the single-core figure, the reference arm.
mkdir -p gpurun_out/r02
python -m paper_2503_16422_b200.build --force > gpurun_out/r02/build.log 2>&1
python bench.py --cpu-single-core > gpurun_out/r02/bench_c3.json 2> gpurun_out/r02/bench_c3.err
python bench.py --config c1 --cpu-single-core --steps 400 > gpurun_out/r02/bench_c1.json 2> gpurun_out/r02/bench_c1.err
python bench.py --config c2 --cpu-single-core > gpurun_out/r02/bench_c2.json 2> gpurun_out/r02/bench_c2.err
python bench.py --config c4 --cpu-single-core > gpurun_out/r02/bench_c4_masked.json 2> gpurun_out/r02/bench_c4_masked.err
python bench.py --config c4 --unmasked --no-cpu-baseline > gpurun_out/r02/bench_c4_unmasked.json 2> gpurun_out/r02/bench_c4_unmasked.err
python bench.py --vq 4096 --no-cpu-baseline > gpurun_out/r02/bench_c3_vq.json 2> gpurun_out/r02/bench_c3_vq.err
python bench.py --literal-masks --no-cpu-baseline > gpurun_out/r02/bench_c3_literal.json 2> gpurun_out/r02/bench_c3_literal.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02/bench_reference.json 2> gpurun_out/r02/bench_reference.err
ls -la gpurun_out/r02
