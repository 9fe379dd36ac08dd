#!/bin/bash
# A/B timing of the libfdgs.so variants in tools/variants (names as arguments)
for v in "$@"; do echo -n "$v "; AB_LIB=tools/variants/libfdgs_$v.so python tools/blend_ab.py --reps 7; done
