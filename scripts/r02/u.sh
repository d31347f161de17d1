# r02u: split-K factor sweep on the under-filled pair-kernel shapes (memset + reduce-add)
O=gpurun_out/r02u; mkdir -p $O
V="--variant k1: --variant k2:-DNE_PAIR_KSPLIT=2 --variant k3:-DNE_PAIR_KSPLIT=3 --variant k4:-DNE_PAIR_KSPLIT=4"
timeout 900 python scripts/r02/ab.py $V --case conv_gemm --M 3 --T 4500 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case conv_gemm --M 8 --T 1000 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case c3p_gemm --M 8 --T 2048 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case c3p_gemm --M 3 --T 2048 >> $O/ab.txt 2>&1
echo done
