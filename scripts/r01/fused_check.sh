cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "scatter or fused_exchange or c5" 2>&1 | tail -4
for ex in nccl fused; do timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 --exchange $ex 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c5', '$ex', d['ms_per_step'], d['roofline']['frac'], d['stages_ms'], d['correctness'])"; done
