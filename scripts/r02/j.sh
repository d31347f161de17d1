# r02j: scale_add_check A/B, op+check tests, C3 fused line, default bench with per-stage event pairs
O=gpurun_out/r02j; mkdir -p $O
timeout 600 python scripts/r02/ab.py --variant new: --variant serial:-DNE_SAC_SERIAL --case c1_sac > $O/ab_sac.txt 2>&1; echo ab rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_w32.py -m gpu -q -k "scale_add or check_fused or c1" > $O/t.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --configs 0 --workload c3 --fuse 1 > $O/b_c3_fused.json 2> $O/b_c3_fused.err; echo fused rc=$?
timeout 900 python bench.py > $O/b_default.json 2> $O/b_default.err; echo default rc=$?
