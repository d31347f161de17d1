# r02z47: bench lines with step_roofline and e2e.link_GBs (default, C3, C3 in order, C4), the bench N > 1 tests
O=gpurun_out/r02z47; mkdir -p $O
timeout 900 python -m pytest tests/test_bench_multirank.py -m gpu -q > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 900 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
run() { name=$1; shift; timeout 600 python bench.py --configs 0 "$@" > $O/b_$name.json 2> $O/b_$name.err; echo $name rc=$?; }
run c3 --workload c3
run c3_inorder --workload c3 --overlap 0
run c4 --workload c4
run c2p_8_4500 --workload c2p --streams 8 --taps 4500 --steps 20
python -c "
import json
for n in ['default','c3','c3_inorder','c4','c2p_8_4500']:
    d=json.load(open('$O/b_'+n+'.json')); print(n, d['value'], d['ms_per_step'], d['step_roofline']['floor_ms'], d['step_roofline']['frac'], d['e2e'].get('link_GBs'))
"
