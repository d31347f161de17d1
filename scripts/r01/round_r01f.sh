# Round-1 pass 6: full GPU suite, every bench line, launch lists and the
# --set full captures the summary/traffic need (each ncu only after its
# command exited 0 without ncu).
mkdir -p gpurun_out/r01f
O=gpurun_out/r01f
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
run() { name=$1; shift; timeout 400 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name rc=$?; }
run c3 --workload c3
run c3_fused --workload c3 --fuse 1
run c3_abft --workload c3 --scheme abft
run c3_base256 --workload c3 --limbs base256
run c3_imad --workload c3 --algo imad --steps 3
run c2 --workload c2
run c2_tc --workload c2 --conv tc
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
run c2p_3_100 --workload c2p --streams 3 --taps 100 --steps 20
run c2p_direct --workload c2p --conv direct --streams 8 --taps 4500 --steps 3
run c1 --workload c1
run c4 --workload c4
run c5 --workload c5 --steps 10
BP="python bench.py --workload c2p --streams 8 --taps 4500 --steps 2 --warmup 3"
B3="python bench.py --workload c3 --steps 2 --warmup 3"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3.csv $B3 > $O/ncu_l3.log 2>&1; echo c3 launches rc=$?
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c2p.csv $BP > $O/ncu_lp.log 2>&1; echo c2p launches rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_entangle_conv_planes|k_conv_prep" -s 3 -c 3 -o $O/prof_c2p $BP > $O/ncu_fp.log 2>&1; echo c2p full rc=$?
