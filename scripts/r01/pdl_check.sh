# Experiment record: measured programmatic dependent launch (reverted).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_w32.py -q -x -k "entangle or scale_add or disentangle or recover or c1 or check" 2>&1 | tail -2
for a in c1 c1 c2 c3; do timeout 300 python bench.py --workload $a --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$a', d['ms_per_step'], d['stages_ms'])"; done
