# r02a: the new parity tests on the timed path, smoke, one default bench line
O=gpurun_out/r02a; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c3_full or c5_full or pair or smoke" > $O/t1.log 2>&1; echo t1 rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo bench rc=$?
timeout 400 python bench.py --workload c5 --steps 5 > $O/bench_c5.json 2> $O/bench_c5.err; echo c5 rc=$?
timeout 300 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1 rc=$?
timeout 300 python bench.py --workload c4 --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4 rc=$?
timeout 300 python bench.py --workload c2 > $O/bench_c2.json 2> $O/bench_c2.err; echo c2 rc=$?
