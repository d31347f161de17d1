"""Time ne_gemm_prep_b at the C3 and C5 sizes (B int32 K x cols -> Bt int8)."""
import torch

import paper_1604_04740_b200 as ne

for K, cols in ((4096, 4096), (16384, 16384), (16384 - 64, 16384)):
    B = torch.randint(-100, 100, (K * cols,), dtype=torch.int32, device="cuda")
    Bt = torch.empty(cols * K, dtype=torch.int8, device="cuda")
    for _ in range(3):
        ne.ne_gemm_prep_b(B, K, cols, Bt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ne.ne_gemm_prep_b(B, K, cols, Bt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"prep_b K={K} cols={cols}: {ms:.4f} ms, {K * cols * 5 / ms / 1e6:.0f} GB/s")
