# Experiment: pair Toeplitz conv at T = 1000 / 300 (Kpad 1280 / 640).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for P in 0 1 0 1; do
  if [ $P = 0 ]; then unset NE_CONV_PAIR; else export NE_CONV_PAIR=1; fi
  for T in 1000 300; do
    timeout 300 python bench.py --workload c2p --streams 8 --taps $T --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('pair=$P T=$T', d['ms_per_step'], d['stages_ms']['conv'])"
  done
done
