# r02z29: C4 x gathers through L2 only (ld.global.cg / L1::no_allocate) and smaller windows, own and shared-atomic reduce
O=gpurun_out/r02z29; mkdir -p $O
timeout 1500 python scripts/r02/ab.py --variant "old:-DNE_PB_OWN_OFF" --variant 'old_cg:-DNE_PB_OWN_OFF -DNE_PB_XLD="ld.global.cg.v4.u64"' \
  --variant 'old_na:-DNE_PB_OWN_OFF -DNE_PB_XLD="ld.global.L1::no_allocate.v4.u64"' \
  --variant 'own_cg:-DNE_PB_XLD="ld.global.cg.v4.u64"' --variant 'old_cg16:-DNE_PB_OWN_OFF -DNE_PB_XLD="ld.global.cg.v4.u64" -DNE_PB_WINDOW_MB=16' \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -12
