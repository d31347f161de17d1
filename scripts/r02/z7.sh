# r02z7: C4 as a bucketed scatter-reduce: parity, then the C4 line both ways
O=gpurun_out/r02z7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "permute_inner" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
timeout 600 python bench.py --configs 0 --workload c4 --steps 5 > $O/b_gather.json 2> $O/b_gather.err; echo bg rc=$?
timeout 600 python bench.py --configs 0 --workload c4 --c4algo bucket --steps 5 > $O/b_bucket.json 2> $O/b_bucket.err; echo bb rc=$?
tail -3 $O/b_bucket.err
