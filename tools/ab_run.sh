#!/bin/bash
# A/B timing of the libfdgs.so variants in tools/variants (names as arguments;
# NAME:ENV=VAL runs variant NAME with an extra environment variable)
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [[ "$spec" == *:* ]] && envs=${spec#*:}
  echo -n "$spec "; env $envs AB_LIB=tools/variants/libfdgs_$v.so python tools/blend_ab.py --reps 7
done
