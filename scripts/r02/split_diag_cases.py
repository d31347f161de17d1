"""Case builders shared by split_diag.py / split_ncu.py (experiments)."""
import torch

import paper_1604_04740_b200 as ne


def conv_case(M, T):
    N = 10 ** 6
    cfg = ne.ne_config_for(M)
    L, b = ne.ne_gemm_limb_plan(cfg, 127)
    bw, kp, plen = ne.ne_conv_geometry(N, T, L)
    c = [torch.randint(-128, 128, (N,), dtype=torch.int32, device='cuda') for _ in range(M)]
    planes = torch.empty(M * L * plen, dtype=torch.int8, device='cuda')
    g = torch.randint(-128, 128, (T,), dtype=torch.int32, device='cuda')
    Gt = torch.empty(bw * kp, dtype=torch.int8, device='cuda')
    ne.ne_entangle_limbs_conv(cfg, c, T, 0, L, planes, None, b, bw)
    ne.ne_conv_prep_taps(g, 0, Gt, None, bw)
    out = [torch.empty(N, dtype=torch.int64, device='cuda') for _ in range(M)]
    return (lambda: ne.ne_op_conv_limbs(cfg, planes, L, Gt, N, T, 0, out, b, bw)), out


def gemm_case(M, R, Cc, K):
    cfg = ne.ne_config_for(M)
    L, b = ne.ne_gemm_limb_plan(cfg, 64)
    A = [torch.randint(-64, 64, (R * K,), dtype=torch.int32, device='cuda') for _ in range(M)]
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device='cuda')
    ne.ne_entangle_limbs(cfg, A, L, planes, None, b)
    Bt = torch.randint(-64, 64, (Cc * K,), dtype=torch.int8, device='cuda')
    out = [torch.empty(R * Cc, dtype=torch.int64, device='cuda') for _ in range(M)]
    return (lambda: ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, b)), out
