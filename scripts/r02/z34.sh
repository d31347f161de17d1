# r02z34: C4 owned-run default: bench line, launch list of the C4 step (DRAM bytes per kernel), ncu --set full of scatter + reduce
O=gpurun_out/r02z34; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
B4="python bench.py --configs 0 --workload c4 --steps 2 --warmup 3"
timeout 400 $B4 > $O/bench_c4.json 2> $O/bench_c4.err; echo b4 rc=$?
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv $B4 > $O/l4.log 2>&1; echo l4 rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_pb_(scatter|reduce)_own" -s 2 -c 2 -o $O/prof_c4own $B4 > $O/f4.log 2>&1; echo f4 rc=$?
