# Experiment record: the NE_GEMM_PAIR hook (k_gemm_pair.cu) — CTA-pair 256 x 128 tiles, double-buffered TMEM.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
NE_GEMM_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm_tc_i8 or pair_digits or zero_padded or c3_full or capped or scatter" 2>&1 | tail -2
for P in 0 1 0 1; do
  if [ $P = 0 ]; then unset NE_GEMM_PAIR; else export NE_GEMM_PAIR=1; fi
  timeout 300 python bench.py --workload c3 --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('pair=$P c3', d['ms_per_step'], d['stages_ms']['gemm'], d['eager_stages_ms']['gemm'], d['correctness'])"
done
export NE_GEMM_PAIR=1
for a in "c3p --streams 8 --kdim 2000" "c5"; do timeout 300 python bench.py --workload $a --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('pair=1 $a', d['ms_per_step'], d['stages_ms'], d['correctness'])"; done
