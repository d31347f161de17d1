# r02f: guard/schedule tests, conv + GEMM parity (pairq entangle, split-K), IMAD tile variants, C2P/C3P lines
O=gpurun_out/r02f; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_guards.py -m gpu -q > $O/t_guards.log 2>&1; echo guards rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "conv or gemm or pair or c3_full" > $O/t_parity.log 2>&1; echo parity rc=$?
for v in 88 84 48 44; do timeout 120 ./scripts/r02/imad_v$v >> $O/imad_variants.txt 2>&1; done; echo variants done
run() { name=$1; shift; timeout 400 python bench.py --configs 0 "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name rc=$?; }
run c2p_3_4500 --workload c2p --streams 3 --taps 4500 --steps 20
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
run c2p_8_1000 --workload c2p --streams 8 --taps 1000 --steps 20
run c3p_8_2000 --workload c3p --streams 8 --kdim 2000 --steps 20
run c3p_3_2000 --workload c3p --streams 3 --kdim 2000 --steps 20
