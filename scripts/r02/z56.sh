# r02z56: final validation of the round's tree: whole GPU suite, smoke, default line
O=gpurun_out/r02z56; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 2700 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
python -c "import json; d=json.load(open('$O/b_default.json')); print(d['value'], d['ms_per_step'], d['stages_ms'], d['roofline']['frac'], d['correctness']['oracle_rows_equal'])"
