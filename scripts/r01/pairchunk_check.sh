# K-chunked limb-major passes on the pair kernel (any K >= 4096).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_limb_major or gemm_tc_i8 or c5 or c3_full or int32_limb or conv_tensor_core" 2>&1 | tail -2
for a in c5 c5 c3; do timeout 300 python bench.py --workload $a --steps 8 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); st=d['stages_ms']; print('$a', d['ms_per_step'], st.get('entangle_gemm', st.get('gemm')), d['correctness'])"; done
