# Round-1 pass 12: launch list and --set full capture of the Toeplitz conv on
# the CTA-pair kernel (C2P M = 8, T = 4500), after the same command exited 0.
mkdir -p gpurun_out/r01l
O=gpurun_out/r01l
NCU=/usr/local/cuda/bin/ncu
BP="python bench.py --workload c2p --streams 8 --taps 4500 --steps 2 --warmup 3"
timeout 300 $BP > $O/bench_c2p.json 2> $O/bench_c2p.err; echo bench rc=$?
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c2p.csv $BP > $O/lp.log 2>&1; echo lp rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_pair|k_entangle_conv_planes|k_conv_tail" -s 3 -c 3 -o $O/prof_c2p $BP > $O/fp.log 2>&1; echo fp rc=$?
