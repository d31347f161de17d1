cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for a in "c3" "c3" "c3 --scheme abft" "c5"; do timeout 300 python bench.py --workload $a --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); st=d['stages_ms']; print('$a', d['ms_per_step'], d['roofline']['frac'], st, d.get('correctness'))"; done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
