# r02z25: C4 owned-run mode with shift-only scatter + block scan and the TMA-staged reduce: tests, A/B, launch list
O=gpurun_out/r02z25; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_guards.py -m gpu -q -x -k "permute or c4 or inner" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
timeout 900 python scripts/r02/ab.py --variant "staged:" --variant "direct:-DNE_PO_DIRECT" --variant "old:-DNE_PB_OWN_OFF" \
  --case c4_permute --T 1 --reps 10 > $O/ab.txt 2>&1; echo ab rc=$?
grep " us$\|failed\|Error" $O/ab.txt | tail -12
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_pb python scripts/r02/c4_once.py > $O/l.csv 2>&1; echo l rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pb_(scatter|reduce)_own" -s 2 -c 2 -o $O/own -f python scripts/r02/c4_once.py > $O/ncu.log 2>&1; echo ncu rc=$?
