cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_w32.py -q -x 2>&1 | tail -3
for w in 64 32; do timeout 600 python bench.py --workload c4 --w $w --steps 5 --warmup 3 2>gpurun_out/c4_$w.err | tail -1 > gpurun_out/c4_$w.json; python -c "import json; d=json.load(open('gpurun_out/c4_$w.json')); print('c4 w=$w', d['ms_per_step'], d['value'], d['roofline']['frac'], d['stages_ms'], d['correctness'])"; done
timeout 600 python bench.py --workload c4 --w 32 --impl reference --steps 1 --warmup 0 2>/dev/null | tail -1 | cut -c1-300
