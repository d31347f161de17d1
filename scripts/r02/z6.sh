# r02z6: does the pair GEMM's epilogue slack absorb a fused check's memory traffic?
# (NE_PAIR_EPI_EXTRA: each CTA reads back its stored delta tile and writes a scratch copy after the drain)
O=gpurun_out/r02z6; mkdir -p $O
timeout 900 python scripts/r02/ab.py --variant base: --variant extra:-DNE_PAIR_EPI_EXTRA --case c3_gemm --reps 30 > $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
