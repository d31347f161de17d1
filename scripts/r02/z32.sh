# r02z32: C4 owned-run defaults (64 MB windows, 896 threads, 4 loads in flight; scatter with 16-byte index stores): tests, A/B, launch list, C4 line
O=gpurun_out/r02z32; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 900 python scripts/r02/ab.py --variant "own:" --variant "old:-DNE_PB_OWN_OFF" --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_pb python scripts/r02/c4_once.py > $O/l.csv 2>&1; echo l rc=$?
timeout 600 python bench.py --configs 0 --workload c4 > $O/b_c4.json 2> $O/b_c4.err; echo c4 rc=$?
