# r02g: A/B of the round-2 schedule changes on one box + ncu of the IMAD.WIDE kernel + GEMM tests
O=gpurun_out/r02g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -k "gemm or pair or c3_full or conv" > $O/t.log 2>&1; echo tests rc=$?
AB="python scripts/r02/ab.py"
timeout 600 $AB --variant split: --variant nosplit:-DNE_PAIR_NO_SPLIT --variant notail:-DNE_PAIR_NO_TAIL --case c3_gemm > $O/ab_c3.txt 2>&1; echo ab1 rc=$?
timeout 600 $AB --variant split: --variant nosplit:-DNE_PAIR_NO_SPLIT --case conv_gemm --M 3 --T 4500 > $O/ab_conv3.txt 2>&1; echo ab2 rc=$?
timeout 600 $AB --variant split: --variant nosplit:-DNE_PAIR_NO_SPLIT --case conv_gemm --M 8 --T 4500 > $O/ab_conv8.txt 2>&1; echo ab3 rc=$?
timeout 600 $AB --variant new: --variant old:-DNE_CONV_ENTANGLE_OLD --case conv_entangle --M 8 --T 4500 > $O/ab_ent8.txt 2>&1; echo ab4 rc=$?
timeout 600 $AB --variant new: --variant old:-DNE_CONV_ENTANGLE_OLD --case conv_entangle --M 3 --T 4500 > $O/ab_ent3.txt 2>&1; echo ab5 rc=$?
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --launch-count 1 --kernel-name regex:imad32w -o $O/imad44 ./scripts/r02/imad_v44 > $O/ncu_imad.log 2>&1; echo ncu rc=$?
timeout 600 python bench.py --configs 0 > $O/bench_c3.json 2> $O/bench_c3.err; echo bench rc=$?
