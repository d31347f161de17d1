cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for M in 8 3; do timeout 300 python bench.py --workload c2p --streams $M --taps 4500 --steps 20 --warmup 5 > gpurun_out/c2p_${M}_4500.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/c2p_${M}_4500.json').read().strip().splitlines()[-1]); print('c2p M=$M', d['ms_per_step'], d['roofline']['frac'], d['stages_ms'])"; done
for M in 8 3; do timeout 300 python bench.py --workload c2p --streams $M --taps 4500 --scheme abft --steps 20 --warmup 5 > gpurun_out/c2p_${M}_4500_abft.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/c2p_${M}_4500_abft.json').read().strip().splitlines()[-1]); print('c2p abft M=$M', d['ms_per_step'], d['stages_ms'])"; done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
