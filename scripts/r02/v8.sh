# r02v8: whole GPU suite (incl. the fuzz cases) + smoke + default bench (C5 overhead in the configs block) + reference arm
O=gpurun_out/r02v8; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
timeout 600 python bench.py --impl reference > $O/b_ref.json 2> $O/b_ref.err; echo ref rc=$?
