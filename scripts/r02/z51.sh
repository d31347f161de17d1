# r02z51: end-of-round validation after the C2 window-load change: whole GPU suite, smoke, default line, reference arm, launch list
O=gpurun_out/r02z51; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 2700 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
cat $O/b_default.json | head -c 600; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/b_ref.json 2> $O/b_ref.err; echo ref rc=$?
head -c 400 $O/b_ref.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 > $O/ncu.log 2>&1; echo ncu rc=$?
