# r02e: whole GPU suite (incl. sanitizers, wide-range GEMM, bench N>1), C4 gather floor + ncu counters,
# IMAD rates, default bench
O=gpurun_out/r02e; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 ./scripts/r02/imad_rate > $O/imad_rate.txt 2>&1; echo imad_rate rc=$?
timeout 300 ./scripts/r02/c4_floor > $O/c4_floor.txt 2>&1; echo c4_floor rc=$?
M1=gpu__time_duration.sum,dram__bytes_read.sum,dram__sectors_read.sum
M2=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum
timeout 600 $NCU --metrics $M1,$M2 --csv ./scripts/r02/c4_floor profile > $O/c4_floor_ncu.csv 2> $O/c4_floor_ncu.err; echo ncu1 rc=$?
if [ $? -ne 0 ] || ! grep -q lts__ $O/c4_floor_ncu.csv; then
  timeout 600 $NCU --metrics $M1 --csv ./scripts/r02/c4_floor profile > $O/c4_floor_ncu_dram.csv 2>> $O/c4_floor_ncu.err; echo ncu1b rc=$?
fi
timeout 600 $NCU --kernel-name regex:k_pinner --launch-count 1 --metrics $M1,$M2 --csv python bench.py --workload c4 --steps 1 --warmup 3 --configs 0 > $O/c4_pinner_ncu.csv 2> $O/c4_pinner_ncu.err; echo ncu2 rc=$?
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench rc=$?
timeout 600 python bench.py --workload c3 --algo imad --steps 3 --configs 0 > $O/bench_imad.json 2> $O/bench_imad.err; echo imad rc=$?
