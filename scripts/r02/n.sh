# r02n: conv-planes entangle, one thread per (stream, quad): A/B + conv tests
O=gpurun_out/r02n; mkdir -p $O
timeout 600 python scripts/r02/ab.py --variant ms: --variant old:-DNE_CONV_ENTANGLE_OLD --case conv_entangle --M 8 --T 4500 > $O/ab8.txt 2>&1; echo ab8 rc=$?
timeout 600 python scripts/r02/ab.py --variant ms: --variant old:-DNE_CONV_ENTANGLE_OLD --case conv_entangle --M 3 --T 4500 > $O/ab3.txt 2>&1; echo ab3 rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -k "conv" > $O/t.log 2>&1; echo t rc=$?
