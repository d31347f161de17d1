# r02z26: C4 owned-run reduce variants (runs walked together R, x loads in flight UN, threads, lockstep lag) vs the shared-atomic reduce
O=gpurun_out/r02z26; mkdir -p $O
timeout 1500 python scripts/r02/ab.py --variant "r4u4:" --variant "r1u8:-DNE_PO_R=1 -DNE_PO_UN=8" --variant "r2u8:-DNE_PO_R=2 -DNE_PO_UN=8" \
  --variant "lag4:-DNE_PO_LAG=4" --variant "t256:-DNE_PO_THREADS=256" --variant "old:-DNE_PB_OWN_OFF" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error" $O/ab.txt | tail -12
