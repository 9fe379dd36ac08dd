python -m paper_2503_16422_b200.build --force > gpurun_out/build.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
for v in "" "--py-submit" "--submit-threads 1" "--submit-threads 6" "--py-submit --sync-compact"; do
  echo "== $v"; python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['host_enqueue'], d['stages_isolated_ms_per_frame'])"
done
