# Experiment record: the NE_GEMM_TILE hook it drives was removed after the measurement.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for T in 0 3 4 0 3 4; do
  if [ $T = 0 ]; then unset NE_GEMM_TILE; else export NE_GEMM_TILE=$T; fi
  python scripts/trace_gemm.py T=$T 2>&1 | grep "clusters=all"
done
