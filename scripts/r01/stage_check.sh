cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for a in "c1" "c2" "c2p --streams 3" "c2p --streams 8" "c3" "c4"; do timeout 600 python bench.py --workload $a --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$a', d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], 'graph', d['stages_ms'], 'eager', d['eager_stages_ms'])"; done
