# r02l: whole GPU suite + smoke + default bench after the schedule clean-up
O=gpurun_out/r02l; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
timeout 600 python bench.py --impl reference > $O/b_reference.json 2> $O/b_reference.err; echo ref rc=$?
