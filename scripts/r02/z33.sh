# r02z33: C4 owned-run scatter chunk / threads
O=gpurun_out/r02z33; mkdir -p $O
timeout 1200 python scripts/r02/ab.py --variant "c4k:" --variant "c8k_t1024:-DNE_PB_CHUNK=8192 -DNE_PB_STHREADS=1024" \
  --variant "c8k_t512:-DNE_PB_CHUNK=8192 -DNE_PB_STHREADS=512" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -6
