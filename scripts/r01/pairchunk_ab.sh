# A/B: C5 per-stream GEMM (K = 16384) on the K-chunked pair kernel vs the single-CTA kernel.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for v in pair single pair single; do
  if [ $v = single ]; then export NE_NO_LONGK_PAIR=1; else unset NE_NO_LONGK_PAIR; fi
  timeout 300 python bench.py --workload c5 --steps 8 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['ms_per_step'], d['stages_ms']['entangle_gemm'], d['clocks']['reasons'])"
done
