for v in np m1 m9 m10; do echo -n "$v "; AB_LIB=tools/variants/libfdgs_$v.so python tools/blend_ab.py --reps 7; done
