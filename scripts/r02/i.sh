# r02i: conv-planes prefetch A/B, whole GPU suite, C2P/C3P/IMAD lines
O=gpurun_out/r02i; mkdir -p $O
AB="python scripts/r02/ab.py"
timeout 600 $AB --variant pf: --variant nopf:-DNE_CONV_PF_OFF --case conv_entangle --M 8 --T 4500 > $O/ab_ent8.txt 2>&1; echo ab1 rc=$?
timeout 600 $AB --variant pf: --variant nopf:-DNE_CONV_PF_OFF --case conv_entangle --M 3 --T 4500 > $O/ab_ent3.txt 2>&1; echo ab2 rc=$?
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
run() { name=$1; shift; timeout 400 python bench.py --configs 0 "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name rc=$?; }
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
run c2p_3_4500 --workload c2p --streams 3 --taps 4500 --steps 20
run c3p_8_2000 --workload c3p --streams 8 --kdim 2000 --steps 20
run c3_imad --workload c3 --algo imad --steps 3
