for v in w8 w16 w32 w8; do for c in c3 c4; do echo -n "$v $c "; AB_LIB=tools/variants/libfdgs_$v.so python tools/blend_ab.py --config $c --frames 12 --reps 5; done; done
