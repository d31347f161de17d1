# r02z46: the widened bucketed permute parity cases (both plans)
O=gpurun_out/r02z46; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "permute_inner_bucketed" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
