# r02p: launch lists + --set full captures (each after its bench command exited 0 without ncu)
O=gpurun_out/r02p; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 120 ./scripts/r02/imad_rate > $O/imad_rate.txt 2>&1; echo imad_rate rc=$?
B3="python bench.py --configs 0 --steps 2 --warmup 3"
timeout 400 $B3 > $O/bench_c3.json 2> $O/bench_c3.err; echo b3 rc=$?
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3.csv $B3 > $O/l3.log 2>&1; echo l3 rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_pair|k_disentangle|k_entangle_pair|k_prep_b" -s 5 -c 5 -o $O/prof_c3 $B3 > $O/f3.log 2>&1; echo f3 rc=$?
B4="python bench.py --configs 0 --workload c4 --steps 2 --warmup 3"
timeout 400 $B4 > $O/bench_c4.json 2> $O/bench_c4.err; echo b4 rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_pinner|k_entangle_aos" -s 2 -c 2 -o $O/prof_c4 $B4 > $O/f4.log 2>&1; echo f4 rc=$?
BI="python bench.py --configs 0 --algo imad --steps 1 --warmup 3"
timeout 400 $BI > $O/bench_imad.json 2> $O/bench_imad.err; echo bi rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"imad32w" -c 1 -o $O/prof_imad $BI > $O/fi.log 2>&1; echo fi rc=$?
B1="python bench.py --configs 0 --workload c1 --n 134217728 --steps 2 --warmup 3"
timeout 400 $B1 > $O/bench_c1.json 2> $O/bench_c1.err; echo b1 rc=$?
timeout 900 $NCU --set full --clock-control none -k regex:"k_scale_add_check|k_entangle|k_disentangle" -s 3 -c 3 -o $O/prof_c1 $B1 > $O/f1.log 2>&1; echo f1 rc=$?
