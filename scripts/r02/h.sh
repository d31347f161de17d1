# r02h: GEMM/conv/guard tests (int32 plain baseline, split-K threshold), IMAD unroll variants, default bench
O=gpurun_out/r02h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -k "gemm or pair or conv or guards" > $O/t.log 2>&1; echo tests rc=$?
for v in 88 44 48; do for u in 1 16; do echo "u=$u" >> $O/imad_variants.txt; timeout 120 ./scripts/r02/imad_v${v}_u$u >> $O/imad_variants.txt 2>&1; done; done; echo variants done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench rc=$?
