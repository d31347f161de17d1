cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "conv" 2>&1 | tail -2
for M in 3 8; do timeout 300 python bench.py --workload c2p --streams $M --taps 4500 --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c2p', $M, d['ms_per_step'], d['roofline']['frac'], d['stages_ms'])"; done
