#!/bin/bash
# Pipelined bench A/B of libfdgs.so variants (tools/variants/libfdgs_NAME.so),
# each copied over the in-tree library in turn: tools/ab_bench.sh STEPS NAME...
steps=$1; shift
cp paper_2503_16422_b200/libfdgs.so /tmp/libfdgs_intree.so
for v in "$@"; do
  cp tools/variants/libfdgs_$v.so paper_2503_16422_b200/libfdgs.so
  echo -n "$v "; timeout 300 python bench.py --steps $steps --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_isolated_ms_per_frame']['blend'])"
done
cp /tmp/libfdgs_intree.so paper_2503_16422_b200/libfdgs.so
