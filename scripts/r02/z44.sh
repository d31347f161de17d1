# r02z44: validation after the conv-planes launch bounds: conv / c2p GPU tests, the whole suite, smoke, C2P lines
O=gpurun_out/r02z44; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
run() { name=$1; shift; timeout 600 python bench.py --configs 0 "$@" > $O/b_$name.json 2> $O/b_$name.err; echo $name rc=$?; }
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
run c2p_3_4500 --workload c2p --streams 3 --taps 4500 --steps 20
run c2p_8_1000 --workload c2p --streams 8 --taps 1000 --steps 20
run c2p_3_100 --workload c2p --streams 3 --taps 100 --steps 20
run c2p_8_4500_abft --workload c2p --streams 8 --taps 4500 --scheme abft --steps 20
run c2p_3_4500_abft --workload c2p --streams 3 --taps 4500 --scheme abft --steps 20
