# r02z50: C2 conv + check with window values of all streams loaded before any store: conv tests, A/B, C2 line
O=gpurun_out/r02z50; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "conv" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
for M in 3 8; do
timeout 600 python scripts/r02/ab.py --variant "wl2:" --variant "wl1:-DNE_CONV_WLOAD2=0" --case c2_conv_check --M $M --T 64 --reps 50 > $O/ab_$M.txt 2>&1; echo ab$M rc=$?
grep " us$\|failed\|Error\|error" $O/ab_$M.txt | tail -3
done
timeout 600 python scripts/r02/ab.py --variant "wl2:" --variant "wl1:-DNE_CONV_WLOAD2=0" --case c2_conv_check --M 3 --T 300 --reps 50 > $O/ab_3_300.txt 2>&1; echo ab300 rc=$?
grep " us$\|failed\|Error\|error" $O/ab_3_300.txt | tail -3
timeout 600 python bench.py --configs 0 --workload c2 > $O/b_c2.json 2> $O/b_c2.err; echo c2 rc=$?
python -c "import json; d=json.load(open('$O/b_c2.json')); print(d['value'], d['ms_per_step'], d['stages_ms'], d['correctness']['oracle_rows_equal'])"
