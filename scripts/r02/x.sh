# r02x: stream-split conv_check (k_conv_check_s): parity, guards, A/B, C2 bench line
O=gpurun_out/r02x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -x -k "conv_check or conv" > $O/t.log 2>&1; echo t rc=$?
tail -2 $O/t.log
timeout 600 python scripts/r02/ab.py --variant one:-DNE_CONV_CHECK_ONE --variant split: --case c2_conv_check --M 3 --T 64 --reps 100 > $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py --variant one:-DNE_CONV_CHECK_ONE --variant split: --case c2_conv_check --M 8 --T 64 --reps 100 >> $O/ab.txt 2>&1
timeout 600 python scripts/r02/ab.py --variant one:-DNE_CONV_CHECK_ONE --variant split: --case c2_conv_check --M 3 --T 1000 --reps 100 >> $O/ab.txt 2>&1
grep " us$\|failed" $O/ab.txt
timeout 600 python bench.py --configs 0 --workload c2 --steps 50 --warmup 5 > $O/b_c2.json 2> $O/b_c2.err; echo b rc=$?
