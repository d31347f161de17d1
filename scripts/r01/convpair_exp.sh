# Experiment: Toeplitz conv on the CTA-pair limb-major kernel (NE_CONV_PAIR=1).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
NE_CONV_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "conv_tensor_core or abft_conv or conv_limbs" 2>&1 | tail -2
for P in 0 1 0 1; do
  if [ $P = 0 ]; then unset NE_CONV_PAIR; else export NE_CONV_PAIR=1; fi
  for M in 8 3; do
    timeout 300 python bench.py --workload c2p --streams $M --taps 4500 --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('pair=$P M=$M', d['ms_per_step'], d['stages_ms']['conv'], d['correctness'])"
  done
done
