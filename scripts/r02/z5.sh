# r02z5: half tiles for the pair kernel's last partial wave: parity + A/B vs HEAD + C3 bench
O=gpurun_out/r02z5; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "pair or c3_full or gemm or conv" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
V="--variant base@HEAD: --variant halves: --variant whole:py:ne.ne_gemm_pair_halves(1)"
timeout 900 python scripts/r02/ab.py $V --case c3_gemm --reps 30 > $O/ab.txt 2>&1
timeout 900 python scripts/r02/ab.py $V --case c3p_gemm --M 8 --T 2048 --reps 30 >> $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
timeout 600 python bench.py --configs 0 --steps 20 --warmup 5 > $O/b_c3.json 2> $O/b_c3.err; echo b rc=$?
