# r02v6: ncu --set full of the pair GEMM whole / forced split 2 / auto split (commit d1b12b3)
O=gpurun_out/r02v6; mkdir -p $O
python scripts/r02/split_ncu.py && echo plain ok
timeout 900 ncu --set full --clock-control none -k regex:k_gemm_pair -c 3 -o $O/split python scripts/r02/split_ncu.py > $O/ncu.log 2>&1; echo ncu rc=$?
tail -5 $O/ncu.log
