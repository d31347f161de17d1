# r02z30: C4 owned-run reduce with L2-only x gathers: loads in flight, threads, flat list, windows, staged vs direct; tests
O=gpurun_out/r02z30; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 1700 python scripts/r02/ab.py --variant "u8:" --variant "u4:-DNE_PO_UN=4" --variant "u4t1024:-DNE_PO_THREADS=1024 -DNE_PO_UN=4" \
  --variant "flat:-DNE_PO_FLAT" --variant "w64:-DNE_PB_WINDOW_MB=64" --variant "direct:-DNE_PO_DIRECT" --variant "r2u8:-DNE_PO_R=2" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -12
