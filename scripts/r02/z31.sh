# r02z31: C4 owned-run reduce: 64 MB windows x threads / loads in flight / lockstep lag
O=gpurun_out/r02z31; mkdir -p $O
timeout 1700 python scripts/r02/ab.py --variant "u8w64:-DNE_PB_WINDOW_MB=64" --variant "t1024u4w64:-DNE_PO_THREADS=1024 -DNE_PO_UN=4 -DNE_PB_WINDOW_MB=64" \
  --variant "t1024u4w64lag1:-DNE_PO_THREADS=1024 -DNE_PO_UN=4 -DNE_PB_WINDOW_MB=64 -DNE_PO_LAG=1" \
  --variant "t768u4w64:-DNE_PO_THREADS=768 -DNE_PO_UN=4 -DNE_PB_WINDOW_MB=64" \
  --variant "t1024u4w48:-DNE_PO_THREADS=1024 -DNE_PO_UN=4 -DNE_PB_WINDOW_MB=48" \
  --variant "t1024u4w64lag3:-DNE_PO_THREADS=1024 -DNE_PO_UN=4 -DNE_PB_WINDOW_MB=64 -DNE_PO_LAG=3" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -12
