# r02z35: validation after the C4 owned-run mode: whole GPU suite, smoke, default bench line, C4 lines, reference arm
O=gpurun_out/r02z35; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
timeout 600 python bench.py --configs 0 --workload c4 > $O/b_c4.json 2> $O/b_c4.err; echo c4 rc=$?
timeout 600 python bench.py --configs 0 --workload c4 --c4algo gather > $O/b_c4_gather.json 2> $O/b_c4_gather.err; echo c4g rc=$?
timeout 600 python bench.py --impl reference > $O/b_ref.json 2> $O/b_ref.err; echo ref rc=$?
