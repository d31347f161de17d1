# r02z55: C3 step with the entangle's planes and prep_b's Bt stored with ordinary (not evict-first) stores
# (NE_KEEP_PLANES), so the GEMM may find them in L2: whole default C3 line A/B, alternating libraries
O=gpurun_out/r02z55; mkdir -p $O
SO=paper_1604_04740_b200/libne.so
python -c "import paper_1604_04740_b200._build as B; B.build(force=True)" > $O/build_base.log 2>&1; echo build rc=$?; cp $SO /tmp/ab_base.so
NE_NVCC_FLAGS="-DNE_KEEP_PLANES=1" python -c "import paper_1604_04740_b200._build as B; B.build(force=True)" > $O/build_keep.log 2>&1; echo build rc=$?; cp $SO /tmp/ab_keep.so
for rep in 1 2 3; do for v in base keep; do
cp /tmp/ab_$v.so $SO
timeout 300 python bench.py --configs 0 --steps 50 > $O/b_${v}_$rep.json 2> $O/b_${v}_$rep.err
python -c "import json; d=json.load(open('$O/b_${v}_$rep.json')); print('$v', d['ms_per_step'], d['stages_ms'], d['correctness']['oracle_rows_equal'], d['clocks']['sm_mhz'])"
done; done
cp /tmp/ab_keep.so $SO
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c3 or pair or entangle or prep" > $O/t.log 2>&1; echo t rc=$?; tail -2 $O/t.log
