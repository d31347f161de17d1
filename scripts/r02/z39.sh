# r02z39: ncu --set full (with source counters) of the C2P conv-planes entangle, M = 8 and M = 3, T = 4500
O=gpurun_out/r02z39; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
for M in 8 3; do
B="python bench.py --configs 0 --workload c2p --streams $M --taps 4500 --steps 2 --warmup 3"
timeout 400 $B > $O/b_$M.json 2> $O/b_$M.err; echo b$M rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_entangle_conv_planes" -s 3 -c 1 -o $O/prof_cp$M -f $B > $O/f$M.log 2>&1; echo f$M rc=$?
done
