# r02v2: A/B of the split-K workspace fix-up vs HEAD (base) and vs forced whole tiles
O=gpurun_out/r02v2; mkdir -p $O
V="--variant base@HEAD: --variant auto: --variant whole:py:ne.ne_gemm_pair_split(1)"
timeout 600 python scripts/r02/ab.py $V --case c3_gemm > $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case conv_gemm --M 3 --T 4500 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case c3p_gemm --M 8 --T 2048 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case conv_gemm --M 8 --T 4500 >> $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
