"""Library reference for the C3 GEMM: cuBLASLt int8 x int8 -> int32 (torch._int_mm)
on the same multiply-adds as the entangled C3 GEMM (3 streams x 2 int8 digits
x 4096^3), timed with CUDA events (L2 holds little of the 0.4 GB outputs)."""
import torch

K = N = 4096
B = torch.randint(-128, 128, (K, N), dtype=torch.int8, device="cuda")
ops = 2 * 6 * 4096 * K * N  # = the C3 tensor work per step (2 digits x 3 streams)
for rows, calls in ((4096, 6), (8192, 3), (24576, 1)):
    A = torch.randint(-128, 128, (rows, K), dtype=torch.int8, device="cuda")
    for _ in range(3):
        C = torch._int_mm(A, B)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        for _ in range(calls):
            C = torch._int_mm(A, B)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLASLt int8 {rows}x{K}x{N} x{calls}: {ms:.4f} ms per C3-equivalent -> {ops / ms / 1e9:.0f} TOP/s")
