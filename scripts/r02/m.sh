# r02m: ncu of the C2P step kernels (conv-planes entangle, taps prep, Toeplitz GEMM, check)
O=gpurun_out/r02m; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
BP="python bench.py --configs 0 --workload c2p --streams 8 --taps 4500 --steps 2 --warmup 3"
timeout 400 $BP > $O/b.json 2> $O/b.err; echo b rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_entangle_conv_planes|k_conv_prep_taps|k_gemm_pair|k_disentangle" -s 4 -c 4 -o $O/prof_c2p $BP > $O/f.log 2>&1; echo f rc=$?
