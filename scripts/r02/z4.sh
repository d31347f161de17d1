# r02z4: pair-tile width 256 vs 128 (NE_PAIR_BN=128: every C3 tile 256 x 128) — the per-tile cost of N = 128 MMAs
O=gpurun_out/r02z4; mkdir -p $O
timeout 900 python scripts/r02/ab.py --variant n256: --variant n128:-DNE_PAIR_BN=128 --case c3_gemm --reps 30 > $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
