# A/B on one box: pair kernel with one accumulators-complete barrier (old) vs
# separate limb-1 / limb-0 barriers (the epilogue holds limb 1 during limb 0's pass).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
run() { for i in 1 2; do timeout 300 python bench.py --workload c3 --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', d['ms_per_step'], d['stages_ms']['gemm'])"; done; }
run new
cp paper_1604_04740_b200/csrc/k_gemm_pair.cu /tmp/new_pair.cu
cp gpurun_old_pair.cu.txt paper_1604_04740_b200/csrc/k_gemm_pair.cu
python -c "from paper_1604_04740_b200._build import build; build(force=True)" > /dev/null 2>&1 || echo build failed
run old
cp /tmp/new_pair.cu paper_1604_04740_b200/csrc/k_gemm_pair.cu
python -c "from paper_1604_04740_b200._build import build; build(force=True)" > /dev/null 2>&1 || echo build failed
run new
