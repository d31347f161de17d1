# r02r: pair-kernel stage count A/B (C3, C2P), conv tests after the conv pair gate change
O=gpurun_out/r02r; mkdir -p $O
AB="python scripts/r02/ab.py"
timeout 900 $AB --variant s6: --variant s5:-DNE_PAIR_STAGES=5 --case c3_gemm > $O/c3.txt 2>&1; echo 1 rc=$?
timeout 900 $AB --variant s6: --variant s5:-DNE_PAIR_STAGES=5 --case c3p_gemm --M 8 --T 2048 > $O/c3p8.txt 2>&1; echo 2 rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -k "conv" > $O/t.log 2>&1; echo t rc=$?
