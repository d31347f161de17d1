# r02z43: C4 owned-run reduce with L2 prefetches of the rows gathered in this window (pf1) or the next (pf2)
O=gpurun_out/r02z43; mkdir -p $O
timeout 900 python scripts/r02/ab.py --variant "pf0:" --variant "pf1:-DNE_PO_PF=1" --variant "pf2:-DNE_PO_PF=2" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -4
