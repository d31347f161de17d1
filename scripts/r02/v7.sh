# r02v7: per-item %globaltimer timeline of the pair kernel (split_trace.py; profiles/r02_split_trace.txt)
O=gpurun_out/r02v7; mkdir -p $O
for a in "c3 1" "c3 0" "conv 1" "conv 0" "conv 2"; do timeout 300 python scripts/r02/split_trace.py $a >> $O/trace.txt 2>&1; done
grep -v "warning\|for (int64\|\^\|detected\|Remark\|^$" $O/trace.txt | tail -150
