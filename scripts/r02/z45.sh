# r02z45: C4 owned-run reduce, the x gather's load flavour: .cg (default) / .nc.L1::no_allocate / .nc / .L1::no_allocate / .lu
O=gpurun_out/r02z45; mkdir -p $O
timeout 1200 python scripts/r02/ab.py --variant "cg:" --variant 'ncna:-DNE_PB_XLD="ld.global.nc.L1::no_allocate.v4.u64"' \
  --variant 'nc:-DNE_PB_XLD="ld.global.nc.v4.u64"' --variant 'na:-DNE_PB_XLD="ld.global.L1::no_allocate.v4.u64"' \
  --variant 'lu:-DNE_PB_XLD="ld.global.lu.v4.u64"' \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -6
