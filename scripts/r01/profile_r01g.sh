# Round-1 pass 7: --set full captures for the kernels whose bench lines lacked
# ncu DRAM traffic (C1 sweep w = 64 / w = 32, C2 fused conv+check, C5 GEMM),
# each only after its bench command exited 0 without ncu.
mkdir -p gpurun_out/r01g
O=gpurun_out/r01g
NCU=/usr/local/cuda/bin/ncu
B1="python bench.py --workload c1 --n 134217728 --steps 2 --warmup 3"
B1W="python bench.py --workload c1 --w 32 --n 134217728 --steps 2 --warmup 3"
B2="python bench.py --workload c2 --steps 2 --warmup 3"
B5="python bench.py --workload c5 --steps 1 --warmup 3"
timeout 300 $B1 > $O/p1.log 2>&1 && timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_entangle<|k_scale_add_check|k_disentangle" -s 6 -c 3 -o $O/prof_c1 $B1 > $O/n1.log 2>&1; echo c1 rc=$?
timeout 300 $B1W > $O/p1w.log 2>&1 && timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_entangle_w32|k_disentangle_w32" -s 6 -c 3 -o $O/prof_c1w $B1W > $O/n1w.log 2>&1; echo c1w rc=$?
timeout 300 $B2 > $O/p2.log 2>&1 && timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_conv_check|k_entangle<|k_disentangle" -s 6 -c 3 -o $O/prof_c2 $B2 > $O/n2.log 2>&1; echo c2 rc=$?
timeout 300 $B5 > $O/p5.log 2>&1 && timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_entangle_limbs_stream" -s 2 -c 2 -o $O/prof_c5 $B5 > $O/n5.log 2>&1; echo c5 rc=$?
