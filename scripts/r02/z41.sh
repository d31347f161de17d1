# r02z41: C2P conv-planes entangle occupancy (min blocks per SM in the launch bounds: registers 76 / 58 / 40 / 32)
O=gpurun_out/r02z41; mkdir -p $O
for M in 8 3; do
timeout 900 python scripts/r02/ab.py --variant "minb1:" --variant "minb4:-DNE_CP_MINB=4" --variant "minb6:-DNE_CP_MINB=6" \
  --variant "minb8:-DNE_CP_MINB=8" --case conv_entangle --M $M --T 4500 --reps 50 > $O/ab_$M.txt 2>&1; echo ab$M rc=$?
grep " us$\|failed\|Error\|error" $O/ab_$M.txt | tail -5
done
