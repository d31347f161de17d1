# r02z24: C4 owned-run mode: launch list and ncu --set full of the scatter and the reduce
O=gpurun_out/r02z24; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 300 python scripts/r02/c4_once.py > $O/once.log 2>&1; echo once rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_pb python scripts/r02/c4_once.py > $O/l.csv 2>&1; echo l rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pb_(scatter|reduce)_own" -s 2 -c 2 -o $O/own -f python scripts/r02/c4_once.py > $O/ncu.log 2>&1; echo ncu rc=$?
