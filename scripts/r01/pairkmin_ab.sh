# Experiment record: NE_PAIR_KMIN hook, removed after the measurement.
# A/B: the pair kernel at the paper's short-K GEMM shapes (Kp = 2048 / 1024 / 256) vs the single-CTA kernel.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for v in 4096 256 4096 256; do
  export NE_PAIR_KMIN=$v
  for a in "c3p --streams 8 --kdim 2000" "c3p --streams 3 --kdim 2000" "c3p --streams 8 --kdim 1000" "c3p --streams 8 --kdim 200"; do
    timeout 300 python bench.py --workload $a --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('kmin=$v $a', d['ms_per_step'], d['stages_ms']['gemm'], d['correctness']['recover_equals_check'])"
  done
done
