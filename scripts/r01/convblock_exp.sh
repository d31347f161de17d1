# Experiment record: Toeplitz block width 256 vs 128 for C2P (NE_CONV_BLOCK hook in bench.py, removed afterwards).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for B in 256 128 256 128; do
  for M in 3 8; do
    NE_CONV_BLOCK=$B timeout 300 python bench.py --workload c2p --streams $M --taps 4500 --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('W=$B M=$M', d['ms_per_step'], d['stages_ms']['conv'], d['correctness'])"
  done
done
