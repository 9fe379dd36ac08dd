python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1
for c in 8 32; do for v in "" "--py-submit" "--submit-threads 6"; do
  echo "== conn=$c $v"; CUDA_DEVICE_MAX_CONNECTIONS=$c python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['host_enqueue']['vs_device'], d['stages']['blend'])"
done; done
