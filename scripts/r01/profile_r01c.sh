# Round-1 profiling, pass 3: C3 with the base-2^l digit plan (launch list + top kernels)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --workload c3 --steps 3 --warmup 3"
timeout 300 $B > gpurun_out/plain_c3.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_l.log 2>&1; echo launches rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_entangle_digits|k_disentangle" -s 6 -c 4 -o gpurun_out/prof_c3_r01c $B > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
