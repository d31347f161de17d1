"""Seeded shape fuzzing of the tensor-core paths against the oracle (round 2).

The parity suite pins chosen shapes; these cases draw shapes from fixed
seeds over each kernel's whole admissible domain — stream counts, ragged
row / column / K extents, digit plans, the persistent grid capped or not —
so that every dispatch branch (CTA-pair kernel, single-CTA kernel, general
digit plans, Toeplitz conv with its tail) is hit at sizes nobody picked.
Every output is compared with the oracle: in full when the oracle finishes
in well under a second, else on sampled rows in every 32-lane TMEM group
plus a Freivalds identity over the whole output (exact in int64: callers
size the test vector so that no product wraps)."""
import numpy as np
import pytest
import torch

import paper_1604_04740_b200 as ne
from _gpu import dev, empty_streams, to_np, to_streams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    ne.build()
    ne.lib()
    assert torch.cuda.is_available()


def _gemm_case(seed):
    """A random two-digit (pair-plan) or base-256 GEMM shape, seeded."""
    r = np.random.default_rng(1000 + seed)
    M = int(r.choice([3, 4, 5, 8]))
    pair_gate = seed % 3 == 0                    # every third case on the CTA-pair kernel's domain
    if pair_gate:
        R = 256 * int(r.integers(1, 5))
        Cc = 256 * int(r.integers(1, 5))
        K = 128 * int(r.integers(32, 65))        # 4096 .. 8192
    else:
        R = 128 * int(r.integers(1, 9))
        Cc = 128 * int(r.integers(1, 9))
        K = 128 * int(r.integers(1, 33))
    bound = int(r.choice([1, 17, 64, 127, 200, 511]))
    cap = int(r.choice([0, 0, 1, 3]))
    return M, R, Cc, K, bound, cap


def _rows(R):
    """One row in every 32-lane group of every 128-row tile (cycling offsets)."""
    return np.array([128 * i + 32 * q + (5 * i + 9 * q) % 32 for i in range(R // 128) for q in range(4)])


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_gemm_limbs(O, seed):
    """ne_op_gemm_limbs over a seeded shape and plan: the limb plan of the
    drawn bound (two digits of base 2^l when it fits int8, else base-256
    digits), the kernel the dispatch picks, the grid capped at 1 or 3
    clusters / pairs in some cases."""
    M, R, Cc, K, bound, cap = _gemm_case(seed)
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, bound)
    if L > 4:
        pytest.skip("plan wider than the limb GEMM (covered by the digit-plan tests)")
    A = np.stack([O.gen_uniform(2000 + seed, 1, m, -bound, bound + 1, R * K) for m in range(M)])
    A[:, 0], A[:, -1] = bound, -bound
    B = O.gen_uniform(2000 + seed, 2, 0, -128, 128, K * Cc)
    B[0], B[-1] = -128, 127
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, diag, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt, diag)
    out = empty_streams(M, R * Cc)
    if cap:
        ne.ne_gemm_trace(None, cap)
    try:
        ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, limb_bits=b)
        torch.cuda.synchronize()
    finally:
        if cap:
            ne.ne_gemm_trace(None, 0)
    assert ne.diag_read(diag)["range_violations"] == 0
    E = O.entangle(ocfg, A).reshape(M, R, K)
    Bm = B.reshape(K, Cc)
    if M * R * Cc * K <= 1 << 29:
        ref = O.op_gemm(ocfg, E, Bm).reshape(M, -1)
        assert (to_np(out) == ref).all(), (M, R, Cc, K, bound, cap, L, b)
        return
    rows = _rows(R)
    ref = O.op_gemm(ocfg, E[:, rows], Bm)
    got = np.stack([out[m].view(R, Cc)[torch.from_numpy(rows).cuda()].cpu().numpy() for m in range(M)])
    assert (got == ref).all(), (M, R, Cc, K, bound, cap, L, b)
    # exact in int64: |E| <= 511 (2^22 + 1) < 2^31, |(B x)_k| <= Cc 128 2 <= 2^18 (Cc <= 1024),
    # K <= 2^13, so |E (B x)| < 2^62; the same bound holds for out @ x
    x = np.random.default_rng(seed).integers(-2, 2, size=Cc)
    bx = Bm @ x
    for m in range(M):
        assert (out[m].cpu().numpy().reshape(R, Cc) @ x == E[m] @ bx).all(), (m, M, R, Cc, K)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_conv_tensor_core(O, seed):
    """ne_op_conv_limbs (tcgen05 Toeplitz conv / correlation, the pair or
    single-CTA kernel by Kpad, the partial-block tail) over seeded N, T, M,
    bound and direction: every output equal to the oracle's."""
    r = np.random.default_rng(3000 + seed)
    M = int(r.choice([3, 4, 8]))
    N = int(r.integers(1, 40000))
    T = int(r.choice([1, 2, 63, 64, 65, 255, 256, 257, 700, 1500, 3000]))
    correlate = int(r.integers(0, 2))
    bound = int(r.choice([1, 64, 127]))
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, bound)
    c = np.stack([O.gen_uniform(4000 + seed, 1, m, -bound, bound + 1, N) for m in range(M)])
    g = O.gen_uniform(4000 + seed, 2, 0, -128, 128, T)
    bw, kp, plen = ne.ne_conv_geometry(N, T, L)
    planes = torch.empty(M * L * plen, dtype=torch.int8, device="cuda")
    Gt = torch.empty(bw * kp, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs_conv(cfg, to_streams(c), T, correlate, L, planes, diag, limb_bits=b, block=bw)
    ne.ne_conv_prep_taps(dev(g, torch.int32), correlate, Gt, diag, block=bw)
    out = empty_streams(M, N)
    ne.ne_op_conv_limbs(cfg, planes, L, Gt, N, T, correlate, out, limb_bits=b, block=bw)
    torch.cuda.synchronize()
    assert ne.diag_read(diag)["range_violations"] == 0
    ref = O.op_conv(ocfg, O.entangle(ocfg, c), g, bool(correlate))
    assert (to_np(out) == ref).all(), (M, N, T, correlate, bound, bw)


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_gemm_then_check_and_recover(O, seed):
    """The whole C3-type pipeline on a seeded shape: entangle -> limb GEMM ->
    disentangle + check (no flags, d_hat = A B) -> recover without every
    stream r (equal to d_hat)."""
    r = np.random.default_rng(5000 + seed)
    M = int(r.choice([3, 4, 8]))
    R, Cc, K = 128 * int(r.integers(1, 5)), 128 * int(r.integers(1, 5)), 128 * int(r.integers(1, 17))
    bound = int(r.choice([3, 31, 100]))
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, bound)
    A = np.stack([O.gen_uniform(6000 + seed, 1, m, -bound, bound + 1, R * K) for m in range(M)])
    B = O.gen_uniform(6000 + seed, 2, 0, -bound, bound + 1, K * Cc)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    delta = empty_streams(M, R * Cc)
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, delta, limb_bits=b)
    d = empty_streams(M, R * Cc)
    diag = ne.diag_new()
    ne.ne_disentangle_check(cfg, delta, 0, d, None, diag)
    plain = np.stack([(A[m].reshape(R, K) @ B.reshape(K, Cc)).reshape(-1) for m in range(M)])
    assert ne.diag_read(diag)["fault_positions"] == 0
    assert (to_np(d) == plain).all()
    for rr in range(M):
        rec = empty_streams(M, R * Cc)
        ne.ne_recover(cfg, [None if m == rr else delta[m] for m in range(M)], rr, rec)
        assert (to_np(rec) == plain).all(), rr


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_permute_inner_bucketed(O, seed):
    """The partitioned scatter-reduce form of the C4 op over seeded n, M,
    block, vlen and value ranges (wide values take its 64-bit path): delta and
    d_hat equal to the oracle's gather + blocked inner product + check."""
    r = np.random.default_rng(7000 + seed)
    M = int(r.choice([3, 4, 5, 8]))
    N = int(r.integers(1, 300000))
    B = int(r.choice([1, 7, 64, 1000, 1024, 3000]))
    vlen = B if r.integers(0, 2) else int(r.integers(1, 2000))
    lim = int(r.choice([2 ** 5, 2 ** 12, 2 ** 20]))
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = np.stack([O.gen_uniform(8000 + seed, 1, m, -lim, lim, N) for m in range(M)])
    perm = O.gen_perm(8000 + seed, 6, N)
    v = O.gen_uniform(8000 + seed, 7, 0, -lim, lim, vlen)
    eps = O.entangle(ocfg, c)
    nb = (N + B - 1) // B
    # the oracle's definition, term by term (products mod 2^64 as the int64 sums of the op)
    xs = np.ascontiguousarray(eps[:, perm].astype(np.int64)).view(np.uint64)
    vs = np.ascontiguousarray(v[np.arange(N) % vlen].astype(np.int64)).view(np.uint64)
    prod = xs * vs
    odelta = np.ascontiguousarray(np.stack([np.add.reduceat(prod[m], np.arange(0, N, B)) for m in range(M)]))
    odelta = odelta.view(np.int64)
    od, _, _ = O.disentangle_check(ocfg, odelta, seed % M)
    ws = torch.empty(ne.ne_permute_inner_workspace(cfg, N, B), dtype=torch.uint8, device="cuda")
    delta, d_out = empty_streams(M, nb), empty_streams(M, nb)
    ne.ne_op_permute_inner_check_bucketed(cfg, dev(eps.T.copy(), torch.int64).reshape(-1), dev(perm, torch.int32),
                                          dev(v, torch.int32), B, seed % M, delta, d_out, ws)
    torch.cuda.synchronize()
    assert (to_np(delta) == odelta).all(), (M, N, B, vlen, lim)
    assert (to_np(d_out) == od).all()
