"""Small launches of the hand-written kernels for compute-sanitizer
(tests/test_gpu_sanitizers.py runs this file under memcheck, racecheck and
synccheck).  Each case also checks its result against the oracle, so a
sanitizer run that silently changes behaviour fails too."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_1604_04740_b200 as ne  # noqa: E402


def streams(a, dt):
    return [torch.from_numpy(np.ascontiguousarray(r)).to(dt).cuda() for r in a]


def host(ts):
    return np.stack([t.cpu().numpy().astype(np.int64) for t in ts])


def empty(M, n):
    return [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(M)]


def gemm_case(M, L, b, R, Cc, K, bound, kernel, fused=False):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    A = np.stack([O.gen_uniform(7, 4, m, -bound, bound + 1, R * K) for m in range(M)])
    B = O.gen_uniform(7, 5, 0, -128, 128, K * Cc)
    assert ne.ne_gemm_kernel_for(cfg, L, b, R, Cc, K) == kernel
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    if L == 1:
        ne.ne_to_limbs(streams(A, torch.int32), 1, planes)
    else:
        ne.ne_entangle_limbs(cfg, streams(A, torch.int32), L, planes, None, b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(torch.from_numpy(B).to(torch.int32).cuda(), K, Cc, Bt)
    out = empty(M, R * Cc)
    E = A if L == 1 else O.entangle(ocfg, A)
    ref = O.op_gemm(ocfg, E.reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    if fused:
        dout = empty(M, R * Cc)
        cnt = torch.zeros(ne.ne_gemm_check_workspace(R, Cc) // 4, dtype=torch.int32, device="cuda")
        diag = ne.diag_new()
        ne.ne_op_gemm_limbs_check(cfg, planes, L, Bt, R, Cc, K, out, 0, dout, cnt, None, diag, b)
        assert (host(dout) == (A.reshape(M, R, K) @ B.reshape(K, Cc)).reshape(M, -1)).all()
        assert ne.diag_read(diag)["fault_positions"] == 0
    else:
        ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, b)
    assert (host(out) == ref).all()


def case_pair():
    gemm_case(3, 2, 22, 256, 512, 4096, 127, "pair")


def case_pair1():
    ne.ne_gemm_trace(None, 2)   # 2 pairs walk all 64 one-digit tiles (both TMEM halves reused)
    try:
        gemm_case(4, 1, 8, 1024, 1024, 1024, 127, "pair")
    finally:
        ne.ne_gemm_trace(None, 0)


def case_tc():
    gemm_case(3, 4, 8, 256, 256, 256, 500, "cta")
    gemm_case(3, 2, 22, 256, 512, 512, 64, "cta")


def case_tc_check():
    gemm_case(3, 2, 22, 256, 512, 256, 64, "cta", fused=True)


def case_scatter():
    M, R, Cc, K, nd = 8, 512, 256, 256, 4
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, 32)
    A = np.stack([O.gen_uniform(8, 4, m, -32, 32, R * K) for m in range(M)])
    B = O.gen_uniform(8, 5, 0, -32, 32, K * Cc)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(torch.from_numpy(B).to(torch.int32).cuda(), K, Cc, Bt)
    As = streams(A, torch.int32)
    planes = torch.empty(L * R * K, dtype=torch.int8, device="cuda")
    chunk = R // nd * Cc
    recv = [torch.empty(M * chunk, dtype=torch.int64, device="cuda") for _ in range(nd)]
    local = torch.empty(R * Cc, dtype=torch.int64, device="cuda")
    ref = O.op_gemm(ocfg, O.entangle(ocfg, A).reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    for m in range(M):
        ne.ne_entangle_limbs_stream(cfg, m, As[m], As[(m - 1) % M], L, planes, None, b)
        ne.ne_op_gemm_limbs_scatter(cfg, planes, L, Bt, R, Cc, K, [w[m * chunk:(m + 1) * chunk] for w in recv], b,
                                    local=local)
        assert (local.cpu().numpy() == ref[m]).all()
    for j in range(nd):
        assert (recv[j].view(M, chunk).cpu().numpy() == ref[:, j * chunk:(j + 1) * chunk]).all()


def case_check():
    for M in (3, 4, 8):
        cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
        n = 4096 + 40
        c = np.stack([O.gen_uniform(9, 1, m, -1000, 1000, n) for m in range(M)])
        eps = O.entangle(ocfg, c)
        eps[1, 77] ^= 1 << 33
        d, bm, diag = empty(M, n), torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda"), ne.diag_new()
        ne.ne_disentangle_check(cfg, streams(eps, torch.int64), 0, d, bm, diag)
        od, flags, nf = O.disentangle_check(ocfg, eps, 0)
        assert (host(d) == od).all() and ne.diag_read(diag)["fault_positions"] == nf == 1
        rec = empty(M, n)
        es = streams(eps, torch.int64)
        ne.ne_recover(cfg, [None] + es[1:], 0, rec)
        assert (host(rec) == O.recover(ocfg, [None] + list(eps[1:]), 0)).all()


def case_pinner():
    M, n, Bk = 4, 1 << 16, 1024
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = np.stack([O.gen_uniform(10, 1, m, -4096, 4096, n) for m in range(M)])
    perm = O.gen_perm(10, 6, n)
    v = O.gen_uniform(10, 7, 0, -4096, 4096, Bk)
    aos = torch.empty(n * M, dtype=torch.int64, device="cuda")
    ne.ne_entangle_aos(cfg, streams(c, torch.int32), aos)
    d = empty(M, n // Bk)
    bm = torch.empty(n // Bk // 32, dtype=torch.int32, device="cuda")
    ne.ne_op_permute_inner_check(cfg, torch.from_numpy(v).to(torch.int32).cuda(), Bk, 0, d, x_aos=aos,
                                 perm=torch.from_numpy(perm).to(torch.int32).cuda(), n=n, bitmap=bm)
    assert (host(d) == O.op_inner(ocfg, c[:, perm], v, Bk)).all()
    eps = O.entangle(ocfg, c)
    out = torch.empty(n // Bk, dtype=torch.int64, device="cuda")
    ne.ne_op_permute_inner_stream(cfg, torch.from_numpy(eps[2].copy()).cuda(), torch.from_numpy(perm).to(torch.int32).cuda(),
                                  torch.from_numpy(v).to(torch.int32).cuda(), Bk, 0, n // Bk, out)
    assert (out.cpu().numpy() == O.op_inner(ocfg, eps[2:3, perm], v, Bk)[0]).all()


def case_conv():
    M, n, T = 3, 8192 + 72, 64
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = np.stack([O.gen_uniform(11, 1, m, -128, 128, n) for m in range(M)])
    g = O.gen_uniform(11, 3, 0, -128, 128, T)
    e = O.entangle(ocfg, c)
    gd = torch.from_numpy(g).to(torch.int32).cuda()
    out, dout = empty(M, n), empty(M, n)
    ne.ne_op_conv_check(cfg, streams(e, torch.int64), gd, out, 0, dout)
    assert (host(dout) == O.op_conv(ocfg, c, g)).all()
    L, b = ne.ne_gemm_limb_plan(cfg, 127)
    bw, kp, plen = ne.ne_conv_geometry(n, T, L)
    pc = torch.empty(M * L * plen, dtype=torch.int8, device="cuda")
    Gt = torch.empty(bw * kp, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs_conv(cfg, streams(c, torch.int32), T, 0, L, pc, None, b, bw)
    ne.ne_conv_prep_taps(gd, 0, Gt, None, bw)
    outc = empty(M, n)
    ne.ne_op_conv_limbs(cfg, pc, L, Gt, n, T, 0, outc, b, bw)
    assert (host(outc) == O.op_conv(ocfg, e, g)).all()


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    ne.lib()
    for name in (sys.argv[1:] or sorted(CASES)):
        CASES[name]()
        torch.cuda.synchronize()
        print("case", name, "ok", flush=True)
