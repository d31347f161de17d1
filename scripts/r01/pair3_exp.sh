# Experiment: pair limb-major GEMM on the other L=2 shapes (C5 per-stream GEMM, C3P, ABFT checksum GEMM).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for P in 0 1; do
  if [ $P = 0 ]; then unset NE_GEMM_PAIR; else export NE_GEMM_PAIR=1; fi
  for a in "c5" "c3p --streams 8 --kdim 2000" "c3p --streams 3 --kdim 2000" "c3p --streams 8 --kdim 200" "c3 --scheme abft"; do
    timeout 300 python bench.py --workload $a --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); st=d['stages_ms']; print('pair=$P $a', d['ms_per_step'], st.get('gemm', st.get('entangle_gemm')), d.get('correctness'))"
  done
done
