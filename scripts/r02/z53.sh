# r02z53: C3P M = 3, N = 200 (paper's smallest GEMM shape): per-kernel launch list, to see what its 22-us stages are
O=gpurun_out/r02z53; mkdir -p $O
timeout 600 python bench.py --configs 0 --workload c3p --streams 3 --kdim 200 --steps 20 > $O/b.json 2> $O/b.err; echo b rc=$?
python -c "import json; d=json.load(open('$O/b.json')); print(d['ms_per_step'], d['stages_ms'], d['eager_stages_ms'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches.csv python bench.py --configs 0 --workload c3p --streams 3 --kdim 200 --steps 2 --warmup 3 > $O/ncu.log 2>&1; echo ncu rc=$?
