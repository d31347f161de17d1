cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin
O=gpurun_out/fin
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
run() { name=$1; shift; timeout 400 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name rc=$?; }
run default
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
run c2p_3_4500 --workload c2p --streams 3 --taps 4500 --steps 20
run c2p_8_1000 --workload c2p --streams 8 --taps 1000 --steps 20
run c2p_3_100 --workload c2p --streams 3 --taps 100 --steps 20
run c2p_8_4500_abft --workload c2p --streams 8 --taps 4500 --scheme abft --steps 20
run c2p_3_4500_abft --workload c2p --streams 3 --taps 4500 --scheme abft --steps 20
