# pipelined throughput with only the front end / only the blend (FDGS_DEBUG_STAGES)
for m in 3 1 2 3; do echo -n "stages=$m "; FDGS_EXPERIMENT=1 FDGS_DEBUG_STAGES=$m python bench.py --no-cpu-baseline --no-e2e --steps 6 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'])"; done
