# r02 final (3): every bench line of the round after the C4 owned-run mode and the side-by-side stages (profiles/r02_bench_*.json via gpurun_out/r02zz3/), the C3 launch list
O=gpurun_out/r02zz3; mkdir -p $O
run() { name=$1; shift; timeout 600 python bench.py --configs 0 "$@" > $O/b_$name.json 2> $O/b_$name.err; echo $name rc=$?; }
timeout 900 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
run c3 --workload c3
run c3_inorder --workload c3 --overlap 0
run c3_abft --workload c3 --scheme abft
run c3_base256 --workload c3 --limbs base256
run c3_fused --workload c3 --fuse 1
run c3_imad --workload c3 --algo imad --steps 3
run c3_a1023 --workload c3 --abound 1023
run c3_a32767_b255 --workload c3 --abound 32767 --bbound 255
run c2 --workload c2
run c2_unfused --workload c2 --fuse 0
run c2_tc --workload c2 --conv tc
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
run c2p_3_4500 --workload c2p --streams 3 --taps 4500 --steps 20
run c2p_8_1000 --workload c2p --streams 8 --taps 1000 --steps 20
run c2p_3_100 --workload c2p --streams 3 --taps 100 --steps 20
run c2p_8_4500_abft --workload c2p --streams 8 --taps 4500 --scheme abft --steps 20
run c2p_3_4500_abft --workload c2p --streams 3 --taps 4500 --scheme abft --steps 20
run c2p_direct --workload c2p --conv direct --streams 8 --taps 4500 --steps 3
run c1 --workload c1
run c1_w32 --workload c1 --w 32
run c1_n2e27 --workload c1 --n 134217728
run c1_w32_n2e27 --workload c1 --w 32 --n 134217728
run c4 --workload c4
run c4_gather --workload c4 --c4algo gather
run c4_soa --workload c4 --layout soa --steps 10
run c4_w32 --workload c4 --w 32
run c5 --workload c5 --steps 10
run c5_fused --workload c5 --steps 10 --exchange fused
run c3p_8_2000 --workload c3p --streams 8 --kdim 2000 --steps 20
run c3p_3_2000 --workload c3p --streams 3 --kdim 2000 --steps 20
run c3p_8_200 --workload c3p --streams 8 --kdim 200 --steps 20
run c3p_3_200 --workload c3p --streams 3 --kdim 200 --steps 20
NCU=/usr/local/cuda/bin/ncu
B3="python bench.py --configs 0 --steps 2 --warmup 3"
timeout 400 $B3 > $O/bench_c3.json 2> $O/bench_c3.err; echo b3 rc=$?
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3.csv $B3 > $O/l3.log 2>&1; echo l3 rc=$?
