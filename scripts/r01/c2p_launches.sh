cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for M in 3 8; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/c2p_$M.csv python bench.py --workload c2p --streams $M --taps 4500 --steps 2 --warmup 3 > /dev/null 2>&1
done
