# r02z52: C2P conv-planes entangle: one-stream-ahead prefetch (NE_CP_PF) and a one-wave grid (NE_CP_GRID), A/B
O=gpurun_out/r02z52; mkdir -p $O
for M in 8 3; do
timeout 900 python scripts/r02/ab.py --variant "base:" --variant "pf:-DNE_CP_PF=1" --variant "pfgrid:-DNE_CP_PF=1 -DNE_CP_GRID=1" \
  --variant "grid:-DNE_CP_GRID=1" --case conv_entangle --M $M --T 4500 --reps 50 > $O/ab_$M.txt 2>&1; echo ab$M rc=$?
grep " us$\|failed\|Error\|error" $O/ab_$M.txt | tail -5
done
