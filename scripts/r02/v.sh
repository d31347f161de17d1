# r02v: split-K with the workspace fix-up (no memset / reduce-add): parity, then A/B vs HEAD
O=gpurun_out/r02v; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pair or c3_full or conv or gemm_capped" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
V="--variant base@HEAD: --variant auto: --variant whole:py:ne.ne_gemm_pair_split(1)"
timeout 600 python scripts/r02/ab.py $V --case c3_gemm > $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case conv_gemm --M 3 --T 4500 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case c3p_gemm --M 8 --T 2048 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py $V --case conv_gemm --M 8 --T 4500 >> $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
timeout 600 python bench.py --configs 0 --steps 20 --warmup 5 > $O/b_c3.json 2> $O/b_c3.err; echo b rc=$?
