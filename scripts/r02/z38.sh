# r02z38: C4 owned-run scatter with 32-bit chunk math, cached keys and the range check off the hot path: permute tests, A/B vs HEAD
O=gpurun_out/r02z38; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 900 python scripts/r02/ab.py --variant "new:" --variant "base@HEAD:" --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error\|error" $O/ab.txt | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:k_pb_scatter python scripts/r02/c4_once.py > $O/l.csv 2>&1; echo l rc=$?
