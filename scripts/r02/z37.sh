# r02z37: smoke with the partitioned C4 op, C4 full-size test on both forms
O=gpurun_out/r02z37; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
tail -2 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4_full or permute" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
