# r02c: bench N>1 path (share-GPU hook, partitions), default bench with configs block
O=gpurun_out/r02c; mkdir -p $O
timeout 1200 python -m pytest tests/test_bench_multirank.py -m gpu -q -x > $O/t_multi.log 2>&1; echo multi rc=$?
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench rc=$?
