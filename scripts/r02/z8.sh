# r02z8: launch list of the bucketed C4 step (which pass costs what)
O=gpurun_out/r02z8; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --configs 0 --workload c4 --c4algo bucket --steps 1 --warmup 3"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:"k_pb" -c 4 --csv --log-file $O/l.csv $B > $O/l.log 2>&1; echo l rc=$?
tail -3 $O/l.log
