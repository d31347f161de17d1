# r02z42: C3 entangle (k_entangle_pair<3>) occupancy: min blocks per SM 1 (64 regs) / 5 (48) / 6 (40)
O=gpurun_out/r02z42; mkdir -p $O
timeout 900 python scripts/r02/ab.py --variant "minb1:" --variant "minb5:-DNE_EP_MINB=5" --variant "minb6:-DNE_EP_MINB=6" \
  --case c3_entangle --reps 50 --flush > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -4
