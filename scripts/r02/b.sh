# r02b: GEMM/ABFT tests incl. the one-digit pair mode; the default bench (C3 + configs block)
O=gpurun_out/r02b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gemm or abft or c3_full" > $O/t1.log 2>&1; echo t1 rc=$?
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench rc=$?
timeout 300 python bench.py --workload c3 --scheme abft --configs 0 > $O/bench_abft.json 2> $O/bench_abft.err; echo abft rc=$?
