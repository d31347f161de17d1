# Round-1 profiling recipe (run on the GPU box via gpurun): smoke, launch lists, ncu --set full captures.
mkdir -p gpurun_out
set -x
NCU=/usr/local/cuda/bin/ncu
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
B="python bench.py --workload c3 --steps 3 --warmup 3"
timeout 300 $B > gpurun_out/plain_c3.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_c3.log 2>&1; echo launches rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 2 -c 1 -o gpurun_out/prof_c3_gemm $B > gpurun_out/ncu_c3_gemm.log 2>&1; echo gemm rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_disentangle -s 2 -c 1 -o gpurun_out/prof_c3_check $B > gpurun_out/ncu_c3_check.log 2>&1; echo check rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_entangle -s 2 -c 1 -o gpurun_out/prof_c3_entangle $B > gpurun_out/ncu_c3_ent.log 2>&1; echo ent rc=$?
B4="python bench.py --workload c4 --steps 3 --warmup 3"
timeout 300 $B4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_pinner -s 2 -c 1 -o gpurun_out/prof_c4_pinner $B4 > gpurun_out/ncu_c4.log 2>&1; echo c4 rc=$?
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c4.csv $B4 > gpurun_out/ncu_c4_l.log 2>&1; echo c4l rc=$?
