# Experiment record: the NE_GEMM_TILE hook it drives was removed after the measurement.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for T in 0 1 2; do
  if [ $T = 0 ]; then unset NE_GEMM_TILE; else export NE_GEMM_TILE=$T; fi
  for a in "c3" "c3p --streams 8 --kdim 2000" "c3p --streams 3 --kdim 2000" "c3p --streams 8 --kdim 200"; do
    timeout 300 python bench.py --workload $a --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('T=$T', '$a', d['ms_per_step'], 'gemm', d['stages_ms']['gemm'], d['roofline']['frac'], d['correctness'])"
  done
done
