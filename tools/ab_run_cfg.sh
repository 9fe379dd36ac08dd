#!/bin/bash
# tools/ab_run.sh for another config: tools/ab_run_cfg.sh CONFIG NAME...
cfg=$1; shift
for v in "$@"; do
  echo -n "$cfg $v "; AB_LIB=tools/variants/libfdgs_$v.so python tools/blend_ab.py --reps 5 --config $cfg
done
