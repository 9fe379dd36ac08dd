#!/bin/bash
python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1
for r in 1 2; do for v in "--py-submit" "--submit-threads 1" "--submit-threads 4" "--submit-threads 4 --max-lead 12" "--submit-threads 6 --max-lead 12" "--submit-threads 6 --max-lead 24" "--submit-threads 2 --max-lead 8"; do
  echo -n "[$v] "; python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages']; print(d['value'], 'blend', s['blend']['share'], 'bin', s['binning']['share'], 'host', d['host_enqueue']['vs_device'])"
done; done
