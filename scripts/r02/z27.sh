# r02z27: C4 owned-run reduce, one list per thread across runs (flat): tests, A/B vs grouped and the shared-atomic reduce
O=gpurun_out/r02z27; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
timeout 1500 python scripts/r02/ab.py --variant "flat8:" --variant "flat4:-DNE_PO_UN=4" --variant "flat4t1024:-DNE_PO_UN=4 -DNE_PO_THREADS=1024" \
  --variant "r1u8:-DNE_PO_GROUPED -DNE_PO_R=1" --variant "old:-DNE_PB_OWN_OFF" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error" $O/ab.txt | tail -12
