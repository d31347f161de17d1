# r02w: persistent prep_b (k_prep_b128p): parity, A/B vs the per-tile grid
O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -x -k "prep_b or c3_full or gemm_pair_limb" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 600 python scripts/r02/ab.py --variant old:-DNE_PREPB_OLD --variant new: --case prep_b --reps 100 > $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
timeout 600 python bench.py --configs 0 --steps 20 --warmup 5 > $O/b_c3.json 2> $O/b_c3.err; echo b rc=$?
