# r02v5: split-K diagnostics after the chained fix-up + pair/conv parity (commit d1b12b3)
O=gpurun_out/r02v5; mkdir -p $O
timeout 600 python scripts/r02/split_diag.py > $O/diag.txt 2>&1; echo rc=$?
cat $O/diag.txt | tail -30
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pair or c3_full or conv or gemm_capped" > $O/t.log 2>&1; echo t rc=$?
tail -3 $O/t.log
