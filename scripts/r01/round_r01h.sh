# Round-1 pass 8: every bench line after the latest kernel changes, launch
# lists of C3 / C2 / C1, and --set full captures of the changed kernels (GEMM
# with 128-byte stages, M=3 four-position disentangle, fused conv+check,
# 256-wide Toeplitz conv, C5 GEMM with row rasterisation); each ncu command
# only after the same bench command exited 0 without ncu.
mkdir -p gpurun_out/r01h
O=gpurun_out/r01h
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
run() { name=$1; shift; timeout 400 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name rc=$?; }
run c3 --workload c3
run c3_fused --workload c3 --fuse 1
run c3_abft --workload c3 --scheme abft
run c3_base256 --workload c3 --limbs base256
run c3_imad --workload c3 --algo imad --steps 3
run c2 --workload c2
run c2_unfused --workload c2 --fuse 0
run c2_tc --workload c2 --conv tc
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
run c2p_3_4500 --workload c2p --streams 3 --taps 4500 --steps 20
run c2p_8_1000 --workload c2p --streams 8 --taps 1000 --steps 20
run c2p_3_100 --workload c2p --streams 3 --taps 100 --steps 20
run c2p_direct --workload c2p --conv direct --streams 8 --taps 4500 --steps 3
run c1 --workload c1
run c1_w32 --workload c1 --w 32
run c1_n2e27 --workload c1 --n 134217728
run c1_w32_n2e27 --workload c1 --w 32 --n 134217728
run c4 --workload c4
run c4_soa --workload c4 --layout soa --steps 10
run c5 --workload c5 --steps 10
B3="python bench.py --workload c3 --steps 2 --warmup 3"
B2="python bench.py --workload c2 --steps 2 --warmup 3"
B1="python bench.py --workload c1 --steps 2 --warmup 3"
BP="python bench.py --workload c2p --streams 8 --taps 4500 --steps 2 --warmup 3"
B5="python bench.py --workload c5 --steps 1 --warmup 3"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3.csv $B3 > $O/l3.log 2>&1; echo l3 rc=$?
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c2.csv $B2 > $O/l2.log 2>&1; echo l2 rc=$?
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c1.csv $B1 > $O/l1.log 2>&1; echo l1 rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_disentangle3x4|k_entangle_pair|k_prep_b" -s 5 -c 5 -o $O/prof_c3 $B3 > $O/f3.log 2>&1; echo f3 rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_conv_check|k_entangle<|k_disentangle" -s 6 -c 3 -o $O/prof_c2 $B2 > $O/f2.log 2>&1; echo f2 rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_entangle_conv_planes" -s 2 -c 2 -o $O/prof_c2p $BP > $O/fp.log 2>&1; echo fp rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_entangle_limbs_stream" -s 2 -c 2 -o $O/prof_c5 $B5 > $O/f5.log 2>&1; echo f5 rc=$?
