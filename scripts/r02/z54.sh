# r02z54: C2P conv-planes entangle, strided-coalesced variant (NE_CP_STRIDED): A/B, then conv/c2p parity with it built in-tree
O=gpurun_out/r02z54; mkdir -p $O
for M in 8 3; do
timeout 900 python scripts/r02/ab.py --variant "base:" --variant "strided:-DNE_CP_STRIDED=1" \
  --case conv_entangle --M $M --T 4500 --reps 50 > $O/ab_$M.txt 2>&1; echo ab$M rc=$?
grep " us$\|failed\|Error\|error" $O/ab_$M.txt | tail -3
done
NE_NVCC_FLAGS="-DNE_CP_STRIDED=1" python -c "import paper_1604_04740_b200._build as B; B.build(force=True)" > $O/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "conv" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
