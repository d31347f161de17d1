# r02z15: partitioned C4 without the count pass (fixed cell capacity + overflow list), parallel window scan
O=gpurun_out/r02z15; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "permute_inner" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
for mb in 32; do
NE_PB_WINDOW_MB=$mb timeout 600 python bench.py --configs 0 --workload c4 --c4algo bucket --steps 3 > $O/b_$mb.json 2> $O/b_$mb.err; echo mb=$mb rc=$?
done
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --configs 0 --workload c4 --c4algo bucket --steps 1 --warmup 3"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:"k_pb" -c 4 --csv --log-file $O/l.csv $B > $O/l.log 2>&1; echo l rc=$?
