# Experiment record: TMA L2 promotion of the operand maps (NE_L2P hook, removed afterwards).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for P in x 0 1 2 x 0 1 2; do
  if [ $P = x ]; then unset NE_L2P; else export NE_L2P=$P; fi
  python scripts/trace_gemm.py L2P=$P 2>&1 | grep "clusters=all"
done
