# r02v4: split-K diagnostics, eager vs graph-replayed (scripts/r02/split_diag.py; commit d1b12b3)
O=gpurun_out/r02v4; mkdir -p $O
timeout 600 python scripts/r02/split_diag.py > $O/diag.txt 2>&1; echo rc=$?
cat $O/diag.txt | tail -30
