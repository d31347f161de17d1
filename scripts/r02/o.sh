# r02o: bench N>1 path at 2 and 4 ranks on one GPU (share-GPU hook)
O=gpurun_out/r02o; mkdir -p $O
timeout 2400 python -m pytest tests/test_bench_multirank.py -m gpu -q > $O/t.log 2>&1; echo t rc=$?
