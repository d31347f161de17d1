# r02q: pair vs single-CTA kernel on the paper's short-K shapes
O=gpurun_out/r02q; mkdir -p $O
AB="python scripts/r02/ab.py"
timeout 900 $AB --variant cta: --variant pair:-DNE_CONV_PAIR_KMIN=1024 --case conv_gemm --M 8 --T 1000 > $O/conv8_1000.txt 2>&1; echo 1 rc=$?
timeout 900 $AB --variant cta: --variant pair:"-DNE_PAIR_KMIN=1024 -DNE_PAIR_TILES_SHORTK=1" --case c3p_gemm --M 3 --T 2048 > $O/c3p3_2048.txt 2>&1; echo 2 rc=$?
timeout 900 $AB --variant pair: --variant cta:"-DNE_PAIR_KMIN=4096 -DNE_PAIR_TILES_SHORTK=1" --case c3p_gemm --M 8 --T 2048 > $O/c3p8_2048.txt 2>&1; echo 3 rc=$?
timeout 900 $AB --variant cta: --variant pair:"-DNE_PAIR_KMIN=1024 -DNE_PAIR_TILES_SHORTK=1" --case c3p_gemm --M 8 --T 1024 > $O/c3p8_1024.txt 2>&1; echo 4 rc=$?
