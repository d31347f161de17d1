# Experiment: 2 x 2 clusters with A and B multicast, NE_GEMM_X2=1.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
NE_GEMM_X2=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm_tc_i8 or pair_digits or zero_padded or c3_full or capped or int32_limb" 2>&1 | tail -2
for T in 0 1 0 1; do
  if [ $T = 0 ]; then unset NE_GEMM_X2; else export NE_GEMM_X2=1; fi
  python scripts/trace_gemm.py X2=$T 2>&1 | grep -v "^$" | head -3
done
for T in 0 1; do
  if [ $T = 0 ]; then unset NE_GEMM_X2; else export NE_GEMM_X2=1; fi
  timeout 300 python bench.py --workload c3 --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('X2=$T c3', d['ms_per_step'], d['stages_ms']['gemm'], d['eager_stages_ms']['gemm'], d['correctness'])"
done
