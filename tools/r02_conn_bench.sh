#!/bin/bash
python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1
for r in 1 2; do for c in 32 8; do for v in "" "--py-submit" "--submit-threads 6"; do
  echo -n "[conn=$c $v] "; CUDA_DEVICE_MAX_CONNECTIONS=$c python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages']; print(d['value'], 'blend', s['blend']['share'], 'bin', s['binning']['share'], 'host', d['host_enqueue']['vs_device'])"
done; done; done
