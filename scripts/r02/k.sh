# r02k: the wide-operand C3 lines (general digit plans on tcgen05), the N=8 row-split GEMM split-K A/B
O=gpurun_out/r02k; mkdir -p $O
run() { name=$1; shift; timeout 600 python bench.py --configs 0 "$@" > $O/b_$name.json 2> $O/b_$name.err; echo $name rc=$?; }
run c3_a1023 --workload c3 --abound 1023
run c3_a32767_b255 --workload c3 --abound 32767 --bbound 255
timeout 600 python scripts/r02/ab.py --variant split: --variant nosplit:-DNE_PAIR_NO_SPLIT --case c3_gemm_rank8 > $O/ab_rank8.txt 2>&1; echo ab rc=$?
