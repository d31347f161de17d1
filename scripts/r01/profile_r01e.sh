# Round-1 profiling, pass 5: C3 (default bench) and the paper-shape convolution (c2p)
# launch lists + --set full captures of their kernels.  Each ncu command runs
# only after the same bench command exited 0 without ncu.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B3="python bench.py --workload c3 --steps 2 --warmup 3"
BP="python bench.py --workload c2p --streams 8 --taps 4500 --steps 2 --warmup 3"
B2="python bench.py --workload c2 --steps 2 --warmup 3"
timeout 300 $B3 > gpurun_out/plain_c3.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv $B3 > gpurun_out/ncu_l3.log 2>&1; echo c3 launches rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_entangle_pair|k_prep_b|k_disentangle" -s 5 -c 5 -o gpurun_out/prof_c3_r01e $B3 > gpurun_out/ncu_f3.log 2>&1; echo c3 full rc=$?
timeout 300 $BP > gpurun_out/plain_c2p.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2p.csv $BP > gpurun_out/ncu_lp.log 2>&1; echo c2p launches rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_entangle_conv_planes" -s 2 -c 2 -o gpurun_out/prof_c2p_r01e $BP > gpurun_out/ncu_fp.log 2>&1; echo c2p full rc=$?
timeout 300 $B2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c2.csv $B2 > gpurun_out/ncu_l2.log 2>&1; echo c2 launches rc=$?
