# r02z3: the paper's conv shapes with 256-output blocks (pair / 128x256 tiles) vs forced 128-output blocks (128x128 tiles)
O=gpurun_out/r02z3; mkdir -p $O
for mt in "3 4500" "8 1000" "3 1000" "8 4500" "3 300"; do set -- $mt
timeout 600 python scripts/r02/ab.py --variant base: --case conv_gemm --M $1 --T $2 --reps 50 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py --variant base: --case conv_gemm128 --M $1 --T $2 --reps 50 >> $O/ab.txt 2>&1
done
grep " us$\|failed" $O/ab.txt
