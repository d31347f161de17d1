# r02y: C5 line with the overhead-vs-plain block
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > $O/b_c5.json 2> $O/b_c5.err; echo b rc=$?
tail -3 $O/b_c5.err
