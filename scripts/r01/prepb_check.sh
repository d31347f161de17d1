cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "prep_b or gemm_tc_i8 or c3_full or pair_digits" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --workload c3 --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3', d['ms_per_step'], d['stages_ms'])"; done
