# r02z10: C4 as a partitioned scatter-reduce (cells = source window x destination range): parity, line, launch list
O=gpurun_out/r02z10; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "permute_inner" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
timeout 600 python bench.py --configs 0 --workload c4 --c4algo bucket --steps 5 > $O/b_bucket.json 2> $O/b_bucket.err; echo bb rc=$?
tail -2 $O/b_bucket.err
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --configs 0 --workload c4 --c4algo bucket --steps 1 --warmup 3"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:"k_pb" -c 4 --csv --log-file $O/l.csv $B > $O/l.log 2>&1; echo l rc=$?
