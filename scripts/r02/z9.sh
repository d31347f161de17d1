# r02z9: bucketed C4, x-window size sweep (NE_PB_WINDOW_MB)
O=gpurun_out/r02z9; mkdir -p $O
for mb in 64 32 16 8 4; do
NE_PB_WINDOW_MB=$mb timeout 600 python bench.py --configs 0 --workload c4 --c4algo bucket --steps 3 > $O/b_$mb.json 2> $O/b_$mb.err; echo mb=$mb rc=$?
done
