"""Memory-safety and race checks of the hand-written kernels without
compute-sanitizer (closed on this GPU pool: runs under it left GPUs needing
a reset).  Instead (SURVEY §5's sanitizer line, done with our own checks):

* out-of-bounds writes: every output buffer of every launch sits between two
  4 KiB guard regions filled with a seeded canary pattern; after the launch
  the guards must be byte-identical (a write one element past either end of
  any output — planes, delta, d_hat, bitmaps, block sums — is caught);
* races and ordering bugs in the mbarrier / TMA / TMEM pipelines, the
  cross-CTA counters of the fused check and the reduce-add multi-launch
  digit plans: launches are repeated with different
  persistent-grid caps (different tile-to-SM schedules) and must give
  bit-identical outputs, each equal to the oracle.

The kernels: k_gemm_pair (two digits, one digit), k_gemm_tc (L = 4,
2; fused check; scatter; multi-launch plans with reduce-add), the entangle
kernels (limbs, pair, split, stream, AoS, conv planes), k_prep_b / k_prep_b_planes, k_disentangle / k_disentangle3x4 + bitmap,
recovery, k_pinner and k_pinner_stream, the direct and Toeplitz convs."""
import numpy as np
import pytest
import torch

import paper_1604_04740_b200 as ne
from _gpu import dev, to_np, to_streams

pytestmark = pytest.mark.gpu
G = 4096  # guard bytes on each side


class Guarded:
    """A device buffer of n elements between two canary regions."""

    def __init__(self, n, dtype, seed):
        esz = torch.tensor([], dtype=dtype).element_size()
        self.g = G // esz
        self.raw = torch.empty(n + 2 * self.g, dtype=dtype, device="cuda")
        bytes_ = self.raw.view(torch.uint8)
        gen = torch.Generator(device="cpu").manual_seed(seed)
        self.canary = torch.randint(0, 256, (bytes_.numel(),), dtype=torch.uint8, generator=gen)
        bytes_.copy_(self.canary.cuda())
        self.t = self.raw[self.g:self.g + n]
        assert self.t.data_ptr() % 16 == 0

    def intact(self):
        b = self.raw.view(torch.uint8).cpu()
        return bool(torch.equal(b[:G], self.canary[:G]) and torch.equal(b[-G:], self.canary[-G:]))


def guarded(M, n, dtype=torch.int64, seed=0):
    return [Guarded(n, dtype, seed * 131 + m) for m in range(M)]


def inner(gs):
    return [g.t for g in gs]


def all_intact(*groups):
    return all(g.intact() for grp in groups for g in (grp if isinstance(grp, list) else [grp]))


def gen(O, seed, tag, M, N, lo, hi):
    return np.stack([O.gen_uniform(seed, tag, m, lo, hi, N) for m in range(M)])


@pytest.mark.parametrize("M,L,bound,R,Cc,K", [
    (3, 2, 127, 256, 512, 4096),    # pair kernel, 6 tiles
    (3, 2, 127, 1024, 1024, 4096),  # pair kernel, 48 tiles
    (4, 1, 127, 1024, 1024, 1024),  # pair kernel, one digit
    (3, 4, 500, 256, 256, 256),     # single CTA, L = 4
    (3, 2, 64, 256, 384, 512),      # single CTA, L = 2, 384 columns
])
def test_gemm_guards_and_schedules(O, M, L, bound, R, Cc, K):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    b = cfg.l if (L == 2 and bound <= 127) else 8
    A = gen(O, 30, 4, M, R * K, -bound, bound + 1)
    B = O.gen_uniform(30, 5, 0, -128, 128, K * Cc)
    P = Guarded(M * L * R * K, torch.int8, 1)
    if L == 1:
        ne.ne_to_limbs(to_streams(A), 1, P.t)
    else:
        ne.ne_entangle_limbs(cfg, to_streams(A), L, P.t, None, b)
    Bt = Guarded(Cc * K, torch.int8, 2)
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt.t)
    E = A if L == 1 else O.entangle(ocfg, A)
    rows = np.arange(0, R, 37)
    ref = O.op_gemm(ocfg, E.reshape(M, R, K)[:, rows], B.reshape(K, Cc))
    x = np.random.default_rng(3).integers(-2, 2, size=Cc)
    bx = B.reshape(K, Cc) @ x
    first = None
    for cap in (0, 1, 3):
        out = guarded(M, R * Cc, seed=cap + 7)
        ne.ne_gemm_trace(None, cap)
        try:
            ne.ne_op_gemm_limbs(cfg, P.t, L, Bt.t, R, Cc, K, inner(out), b)
            torch.cuda.synchronize()
        finally:
            ne.ne_gemm_trace(None, 0)
        assert all_intact(out, P, Bt), cap
        got = to_np(inner(out))
        if first is None:
            first = got
            assert (got.reshape(M, R, Cc)[:, rows] == ref).all()
            for m in range(M):
                assert (got[m].reshape(R, Cc) @ x == E.reshape(M, R, K)[m] @ bx).all()
        assert (got == first).all(), cap   # every schedule: bit-identical


def test_fused_check_and_scatter_guards(O):
    M, R, Cc, K = 3, 256, 512, 256
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, 64)
    A = gen(O, 31, 4, M, R * K, -64, 65)
    B = O.gen_uniform(31, 5, 0, -64, 64, K * Cc)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, None, b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    plain = (A.reshape(M, R, K) @ B.reshape(K, Cc)).reshape(M, -1)
    outs = []
    for rep in range(3):
        delta, dout = guarded(M, R * Cc, seed=10 + rep), guarded(M, R * Cc, seed=20 + rep)
        bm = Guarded(R * Cc // 32, torch.int32, 30 + rep)
        cnt = torch.zeros(ne.ne_gemm_check_workspace(R, Cc) // 4, dtype=torch.int32, device="cuda")
        diag = ne.diag_new()
        ne.ne_op_gemm_limbs_check(cfg, planes, L, Bt, R, Cc, K, inner(delta), 0, inner(dout), cnt, bm.t, diag, b)
        torch.cuda.synchronize()
        assert all_intact(delta, dout, bm)
        assert int(cnt.abs().sum()) == 0 and ne.diag_read(diag)["fault_positions"] == 0
        assert (to_np(inner(dout)) == plain).all() and int(bm.t.abs().sum()) == 0
        outs.append(to_np(inner(delta)))
    assert all((o == outs[0]).all() for o in outs)
    # scatter: 4 receivers + the local copy, guarded
    M5, R5 = 8, 512
    cfg5, ocfg5 = ne.ne_config_for(M5), O.config_for(M5, 64)
    L5, b5 = ne.ne_gemm_limb_plan(cfg5, 32)
    A5 = gen(O, 32, 4, M5, R5 * K, -32, 32)
    As = to_streams(A5)
    pm = torch.empty(L5 * R5 * K, dtype=torch.int8, device="cuda")
    chunk = R5 // 4 * Cc
    recv = [Guarded(M5 * chunk, torch.int64, 40 + j) for j in range(4)]
    loc = Guarded(R5 * Cc, torch.int64, 50)
    ref = O.op_gemm(ocfg5, O.entangle(ocfg5, A5).reshape(M5, R5, K), B.reshape(K, Cc)).reshape(M5, -1)
    for m in range(M5):
        ne.ne_entangle_limbs_stream(cfg5, m, As[m], As[(m - 1) % M5], L5, pm, None, b5)
        ne.ne_op_gemm_limbs_scatter(cfg5, pm, L5, Bt, R5, Cc, K, [r.t[m * chunk:(m + 1) * chunk] for r in recv], b5,
                                    local=loc.t)
        torch.cuda.synchronize()
        assert (loc.t.cpu().numpy() == ref[m]).all()
    assert all_intact(recv, loc)
    for j in range(4):
        assert (recv[j].t.view(M5, chunk).cpu().numpy() == ref[:, j * chunk:(j + 1) * chunk]).all()


@pytest.mark.parametrize("M,a,bb", [(3, 1 << 10, 128), (3, 1 << 15, 1 << 15), (8, 1 << 20, 1 << 10)])
def test_plan_gemm_guards(O, M, a, bb):
    """Split / multi-plane digit plans: entangle, B planes and the
    reduce-add launches write only inside their buffers; two runs agree."""
    R, Cc, K = 128, 256, 256
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    plan = ne.ne_gemm_plan_for(cfg, a, bb)
    A = gen(O, 33, 4, M, R * K, -a, a + 1)
    B = O.gen_uniform(33, 5, 0, -bb, bb + 1, K * Cc)
    P = Guarded(M * plan.LA * R * K, torch.int8, 60)
    ne.ne_entangle_plan(cfg, to_streams(A), plan, P.t)
    Bt = Guarded(plan.LB * Cc * K, torch.int8, 61)
    ne.ne_gemm_prep_b_planes(dev(B, torch.int32), K, Cc, plan.LB, Bt.t)
    ref = O.op_gemm(ocfg, O.entangle(ocfg, A).reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    for rep in range(2):
        out = guarded(M, R * Cc, seed=62 + rep)
        ne.ne_op_gemm_plan(cfg, P.t, plan, Bt.t, R, Cc, K, inner(out))
        torch.cuda.synchronize()
        assert all_intact(out, P, Bt)
        assert (to_np(inner(out)) == ref).all()


@pytest.mark.parametrize("M,N", [(3, 4096 + 40), (4, 1000), (8, 777), (3, 5)])
def test_check_recover_guards(O, M, N):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 34, 1, M, N, -1000, 1000)
    eps = O.entangle(ocfg, c)
    eps[1, N // 2] ^= 1 << 40
    d = guarded(M, N, seed=70)
    bm = Guarded((N + 31) // 32, torch.int32, 71)
    diag = ne.diag_new()
    es = to_streams(eps, torch.int64)
    ne.ne_disentangle_check(cfg, es, 0, inner(d), bm.t, diag)
    od, flags, nf = O.disentangle_check(ocfg, eps, 0)
    assert all_intact(d, bm) and (to_np(inner(d)) == od).all() and ne.diag_read(diag)["fault_positions"] == nf
    for r in range(M):
        rec = guarded(M, N, seed=72 + r)
        ne.ne_recover(cfg, [None if m == r else es[m] for m in range(M)], r, inner(rec))
        assert all_intact(rec)
        assert (to_np(inner(rec)) == O.recover(ocfg, [None if m == r else eps[m] for m in range(M)], r)).all()


def test_entangle_and_gather_guards(O):
    M, n, Bk = 4, 1 << 16, 1024
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 35, 1, M, n, -4096, 4096)
    aos = Guarded(n * M, torch.int64, 80)
    ne.ne_entangle_aos(cfg, to_streams(c), aos.t)
    eps = O.entangle(ocfg, c)
    assert aos.intact() and (aos.t.cpu().numpy().reshape(n, M).T == eps).all()
    perm = O.gen_perm(35, 6, n)
    v = O.gen_uniform(35, 7, 0, -4096, 4096, Bk)
    vd, pd = dev(v, torch.int32), dev(perm, torch.int32)
    d, dl = guarded(M, n // Bk, seed=81), guarded(M, n // Bk, seed=82)
    bm = Guarded(n // Bk // 32, torch.int32, 83)
    ne.ne_op_permute_inner_check(cfg, vd, Bk, 0, inner(d), x_aos=aos.t, perm=pd, n=n, delta_out=inner(dl),
                                 bitmap=bm.t)
    assert all_intact(d, dl, bm) and (to_np(inner(d)) == O.op_inner(ocfg, c[:, perm], v, Bk)).all()
    o1 = Guarded(n // Bk - 3, torch.int64, 84)
    ne.ne_op_permute_inner_stream(cfg, dev(eps[1], torch.int64), pd, vd, Bk, 2, n // Bk - 3, o1.t)
    assert o1.intact()
    assert (o1.t.cpu().numpy() == O.op_inner(ocfg, eps[1:2, perm], v, Bk)[0][2:n // Bk - 1]).all()
    for L, b, bound in ((4, 8, 4096), (2, cfg.l, 127)):   # base-256 and two-digit entangle kernels
        P = Guarded(M * L * n, torch.int8, 85 + L)
        cc = gen(O, 36, 1, M, n, -bound, bound + 1)
        ne.ne_entangle_limbs(cfg, to_streams(cc), L, P.t, None, b)
        p = P.t.cpu().numpy().astype(np.int64).reshape(M, L, n)
        assert P.intact() and (sum(p[:, i] << (b * i) for i in range(L)) == O.entangle(ocfg, cc)).all()


@pytest.mark.parametrize("M,N,T,corr", [(3, 65536, 64, 0), (8, 20000, 1000, 1), (3, 4096, 2, 0),
                                         (4, 8192 + 6, 300, 0)])
def test_conv_guards(O, M, N, T, corr):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 37, 1, M, N, -128, 128)
    g = O.gen_uniform(37, 3, 0, -128, 128, T)
    e = O.entangle(ocfg, c)
    gd = dev(g, torch.int32)
    out, dout = guarded(M, N, seed=90), guarded(M, N, seed=91)
    ne.ne_op_conv_check(cfg, to_streams(e, torch.int64), gd, inner(out), 0, inner(dout), correlate=bool(corr))
    assert all_intact(out, dout) and (to_np(inner(dout)) == O.op_conv(ocfg, c, g, bool(corr))).all()
    L, b = ne.ne_gemm_limb_plan(cfg, 127)
    bw, kp, plen = ne.ne_conv_geometry(N, T, L)
    P = Guarded(M * L * plen, torch.int8, 92)
    Gt = Guarded(bw * kp, torch.int8, 93)
    ne.ne_entangle_limbs_conv(cfg, to_streams(c), T, corr, L, P.t, None, b, bw)
    ne.ne_conv_prep_taps(gd, corr, Gt.t, None, bw)
    res = []
    for rep in range(2):
        o = guarded(M, N, seed=94 + rep)
        ne.ne_op_conv_limbs(cfg, P.t, L, Gt.t, N, T, corr, inner(o), b, bw)
        torch.cuda.synchronize()
        assert all_intact(o, P, Gt)
        res.append(to_np(inner(o)))
    assert (res[0] == O.op_conv(ocfg, e, g, bool(corr))).all() and (res[1] == res[0]).all()
