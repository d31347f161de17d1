# r02d: wide-range GEMM plans, IMAD.WIDE kernel, bench N>1 path (share-GPU hook), IMAD bench
O=gpurun_out/r02d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "wide_range or full_int64 or imad" > $O/t_gemm.log 2>&1; echo gemm rc=$?
timeout 1500 python -m pytest tests/test_bench_multirank.py -m gpu -q -x > $O/t_multi.log 2>&1; echo multi rc=$?
timeout 600 python bench.py --workload c3 --algo imad --steps 3 --configs 0 > $O/bench_imad.json 2> $O/bench_imad.err; echo imad rc=$?
