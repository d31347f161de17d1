# r02s: IMAD.WIDE GEMM with the padded A tile; imad tests; the C3 imad line
O=gpurun_out/r02s; mkdir -p $O
for v in 88 48; do timeout 120 ./scripts/r02/imad_v${v}_pad >> $O/imad_pad.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -k "imad" > $O/t.log 2>&1; echo t rc=$?
timeout 600 python bench.py --configs 0 --workload c3 --algo imad --steps 3 > $O/b_imad.json 2> $O/b_imad.err; echo b rc=$?
