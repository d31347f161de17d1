# r02z18: scatter chunk / thread-count variants of the partitioned C4 stage, and the gather kernel
O=gpurun_out/r02z18; mkdir -p $O
timeout 1500 python scripts/r02/ab.py --variant "c8k_512:" --variant "c4k_256:-DNE_PB_CHUNK=4096 -DNE_PB_STHREADS=256" \
  --variant "c4k_512:-DNE_PB_CHUNK=4096" --variant "c16k_1024:-DNE_PB_CHUNK=16384 -DNE_PB_STHREADS=1024" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py --variant gather: --case c4_permute --T 0 --reps 10 >> $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
