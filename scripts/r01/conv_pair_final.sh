cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_limb_major or conv_tensor_core or abft_conv" 2>&1 | tail -2
for M in 8 3; do timeout 300 python bench.py --workload c2p --streams $M --taps 4500 --steps 20 --warmup 5 > gpurun_out/c2p_${M}_4500.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/c2p_${M}_4500.json').read().strip().splitlines()[-1]); print('c2p M=$M', d['ms_per_step'], d['roofline']['frac'], d['stages_ms']['conv'])"; done
timeout 300 python bench.py --workload c3 --steps 50 --warmup 5 > gpurun_out/c3_final.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/c3_final.json').read().strip().splitlines()[-1]); print('c3', d['ms_per_step'], d['roofline']['frac'], d['stages_ms'])"
