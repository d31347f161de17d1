# r02z28: C4 with a TMA L2 bulk prefetch of the next x window (each CTA its share): own (R=1, UN=8) and shared-atomic reduce, with/without prefetch
O=gpurun_out/r02z28; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
timeout 1500 python scripts/r02/ab.py --variant "own_pf:" --variant "own_nopf:-DNE_PB_PREFETCH=0" \
  --variant "old_pf:-DNE_PB_OWN_OFF" --variant "old_nopf:-DNE_PB_OWN_OFF -DNE_PB_PREFETCH=0" --variant "own_pf_lag4:-DNE_PO_LAG=4" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error" $O/ab.txt | tail -12
