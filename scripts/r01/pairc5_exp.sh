# Experiment record: NE_PAIR_ANYK / NE_PAIR_RASTER hooks, removed after the measurement.
# Experiment: C5's per-stream GEMM (K = 16384) on the pair kernel, raster on / off.
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
for cfg in "x" "1:1" "1:0"; do
  unset NE_PAIR_ANYK NE_PAIR_RASTER
  if [ $cfg != x ]; then export NE_PAIR_ANYK=1; export NE_PAIR_RASTER=${cfg#*:}; fi
  timeout 300 python bench.py --workload c5 --steps 6 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg', d['ms_per_step'], d['stages_ms']['entangle_gemm'], d['correctness'])"
done
