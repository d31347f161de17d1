# r02z19: partitioned C4, one reduce CTA per SM, consecutive pairs combined in registers (U = 8 / 4)
O=gpurun_out/r02z19; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "permute_inner" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 1500 python scripts/r02/ab.py --variant "u8:-DNE_PB_CHUNK=4096" --variant "u4:-DNE_PB_CHUNK=4096 -DNE_PB_U=4" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
