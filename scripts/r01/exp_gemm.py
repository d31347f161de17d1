"""Experiment: where the tcgen05 GEMM time goes (epilogue variants via
NE_GEMM_EPI, per-tile fixed cost via K doubling).  Usage: exp_gemm.py"""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) == 1:
    for epi in ("0", "1", "2"):
        env = dict(os.environ, NE_GEMM_EPI=epi)
        print(subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True).stdout, end="")
    sys.exit(0)
import torch
import paper_1604_04740_b200 as ne
cfg = ne.ne_config_for(3)
for (R, C, K, L) in ((4096, 4096, 4096, 4), (4096, 4096, 8192, 4), (4096, 4096, 4096, 1), (4096, 4096, 4096, 2)):
    planes = torch.randint(-100, 100, (3 * L * R * K,), dtype=torch.int8, device="cuda")
    Bt = torch.randint(-100, 100, (C * K,), dtype=torch.int8, device="cuda")
    out = [torch.empty(R * C, dtype=torch.int64, device="cuda") for _ in range(3)]
    for _ in range(3):
        ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, C, K, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10):
        ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, C, K, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    tops = 2 * L * 3 * R * C * K / ms / 1e9
    print(f"EPI={os.environ.get('NE_GEMM_EPI')} R={R} C={C} K={K} L={L}: {ms:.4f} ms  {tops:.0f} int8 TOP/s")
