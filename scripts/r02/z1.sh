# r02z1: seeded shape fuzzing of the tensor-core paths (tests/test_gpu_fuzz.py)
O=gpurun_out/r02z1; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -rs --durations=10 > $O/t.log 2>&1; echo t rc=$?
tail -25 $O/t.log
