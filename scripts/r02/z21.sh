# r02z21: the fuzz cases of the partitioned C4 op + the whole GPU suite + smoke
O=gpurun_out/r02z21; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x -k "permute" > $O/tf.log 2>&1; echo tf rc=$?
tail -3 $O/tf.log
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
