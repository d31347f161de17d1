# r02z20: C4 default = the partitioned scatter-reduce: tests, both C4 lines, per-kernel DRAM bytes of the stage
O=gpurun_out/r02z20; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 600 python bench.py --configs 0 --workload c4 > $O/b_c4.json 2> $O/b_c4.err; echo b4 rc=$?
timeout 600 python bench.py --configs 0 --workload c4 --c4algo gather > $O/b_c4_gather.json 2> $O/b_c4_gather.err; echo b4g rc=$?
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --configs 0 --workload c4 --steps 1 --warmup 3"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_pb|k_disentangle|k_entangle_aos" -c 12 --csv --log-file $O/l.csv $B > $O/l.log 2>&1; echo l rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_pb_reduce" -s 1 -c 1 -o $O/prof_c4reduce $B > $O/f.log 2>&1; echo f rc=$?
