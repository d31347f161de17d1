# r02z23: C4 owned-run mode (sorted runs + run index, atomic-free reduce): permute tests, A/B vs the shared-atomic reduce, C4 line
O=gpurun_out/r02z23; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
timeout 900 python scripts/r02/ab.py --variant "own:" --variant "old:-DNE_PB_OWN_OFF" --variant "own1024:-DNE_PO_THREADS=1024" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error" $O/ab.txt | tail -12
timeout 600 python bench.py --configs 0 --workload c4 > $O/b_c4.json 2> $O/b_c4.err; echo c4 rc=$?
