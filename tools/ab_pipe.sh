#!/bin/bash
# pipelined bench per libfdgs variant: tools/ab_pipe.sh CONFIG NAME...
c=$1; shift
for v in "$@"; do echo -n "$v $c "; AB_LIB=tools/variants/libfdgs_$v.so python tools/ab_bench.py --config $c; done
