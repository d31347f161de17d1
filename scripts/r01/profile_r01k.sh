# Round-1 pass 11: the CTA-pair limb-major GEMM (k_gemm_pair) — C3 bench lines,
# C3 launch list and a --set full capture of the new kernel; each ncu command
# only after the same bench command exited 0 without ncu.
mkdir -p gpurun_out/r01k
O=gpurun_out/r01k
NCU=/usr/local/cuda/bin/ncu
run() { name=$1; shift; timeout 400 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name rc=$?; }
run c3 --workload c3
run c3_abft --workload c3 --scheme abft
run c3_fused --workload c3 --fuse 1
run c3_base256 --workload c3 --limbs base256
B3="python bench.py --workload c3 --steps 2 --warmup 3"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3.csv $B3 > $O/l3.log 2>&1; echo l3 rc=$?
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"k_gemm_pair" -s 3 -c 1 -o $O/prof_c3pair $B3 > $O/f3.log 2>&1; echo f3 rc=$?
PYTHONPATH=. python scripts/cublas_int8_ref.py > $O/cublas.txt 2>&1; echo cublas rc=$?
