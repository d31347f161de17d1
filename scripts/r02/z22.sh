# r02z22: re-entry validation of HEAD: whole GPU suite + smoke + default bench line
O=gpurun_out/r02z22; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
