# r02z2: C3 entangle, 8 vs 16 positions per thread (NE_ENT_PAIR16), warm and flushed L2
O=gpurun_out/r02z2; mkdir -p $O
timeout 600 python scripts/r02/ab.py --variant p8: --variant p16:-DNE_ENT_PAIR16 --case c3_entangle --reps 50 > $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py --variant p8: --variant p16:-DNE_ENT_PAIR16 --case c3_entangle --reps 50 --flush >> $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
