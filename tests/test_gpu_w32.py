"""GPU parity of the w = 32 container path (the paper's own instantiation,
P:528-530: M = 3, l = 11, k = 10; Table II for other M) against the CPU
oracle, whose arithmetic is generic in w (values reduced mod 2^w).  All
integer: bit-exact."""
import numpy as np
import pytest
import torch

import paper_1604_04740_b200 as ne
from _gpu import bitmap_to_flags, dev, to_np, to_streams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    ne.build()
    ne.lib()
    assert torch.cuda.is_available()


def gen(O, seed, tag, M, N, lo, hi):
    return np.stack([O.gen_uniform(seed, tag, m, lo, hi, N) for m in range(M)])


def empty32(M, N):
    return [torch.empty(N, dtype=torch.int32, device="cuda") for _ in range(M)]


@pytest.mark.parametrize("N", [4096, 4099, 1, 130])
def test_w32_c1_chain(O, N):
    """C1 at w = 32: eps = E c, alpha = E a, delta = 37 eps + alpha (one fused
    pass), disentangle + check for every excluded r, recovery of every r; the
    disentangled result equals 37 c + a (Props 1/3)."""
    M = 3
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    assert (cfg.l, cfg.k) == (11, 10)
    c = gen(O, 0, 1, M, N, -2 ** 10, 2 ** 10)
    a = gen(O, 0, 2, M, N, -2 ** 10, 2 ** 10)
    diag = ne.diag_new()
    eps, alpha = empty32(M, N), empty32(M, N)
    ne.ne_entangle_w32(cfg, to_streams(c), eps, diag)
    ne.ne_entangle_w32(cfg, to_streams(a), alpha, diag)
    E, A = O.entangle(ocfg, c), O.entangle(ocfg, a)
    assert (to_np(eps) == E).all() and (to_np(alpha) == A).all()
    ne.ne_op_scale_add_w32(cfg, eps, 37, None, alpha, 1)
    D = O.op_add(ocfg, O.op_scale(ocfg, E, 37), A, 1)
    assert (to_np(eps) == D).all()
    plain = 37 * c + a
    for r in range(M):
        d_out = empty32(M, N)
        bm = torch.full(((N + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        ne.ne_disentangle_check_w32(cfg, eps, r, d_out, bm, diag)
        ref, flags, nf = O.disentangle_check(ocfg, D, r)
        assert (to_np(d_out) == ref).all() and (ref == plain).all()
        assert (bitmap_to_flags(bm, N) == flags).all() and nf == 0
        rec = empty32(M, N)
        ne.ne_recover_w32(cfg, [None if m == r else eps[m] for m in range(M)], r, rec)
        assert (to_np(rec) == plain).all()
    d = ne.diag_read(diag)
    assert d["range_violations"] == 0 and d["fault_positions"] == 0


@pytest.mark.parametrize("M", [4, 5, 8, 11, 16, 32])
def test_w32_every_M(O, M):
    """Table II configurations: entangle, scale by g[n], add, check and recover
    agree with the oracle at the edges of the dynamic range."""
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    hi = ne.ne_dynamic_range(cfg)
    assert hi == O.dynamic_range(ocfg)
    N = 1000 + M
    c = gen(O, 5, 1, M, N, -hi, hi + 1)
    c[:, 0], c[:, 1] = hi, -hi
    eps = empty32(M, N)
    ne.ne_entangle_w32(cfg, to_streams(c), eps)
    E = O.entangle(ocfg, c)
    assert (to_np(eps) == E).all()
    g = np.ones(N, dtype=np.int64)
    g[::3] = -1
    ne.ne_op_scale_add_w32(cfg, eps, 1, torch.from_numpy(g.astype(np.int32)).cuda())
    D = O.op_scale(ocfg, E, 1, g)
    assert (to_np(eps) == D).all()
    r = M // 2
    d_out = empty32(M, N)
    diag = ne.diag_new()
    ne.ne_disentangle_check_w32(cfg, eps, r, d_out, None, diag)
    ref, _, nf = O.disentangle_check(ocfg, D, r)
    assert (to_np(d_out) == ref).all() and (ref == c * g).all()
    assert ne.diag_read(diag)["fault_positions"] == nf == 0
    rec = empty32(M, N)
    ne.ne_recover_w32(cfg, [None if m == 1 else eps[m] for m in range(M)], 1, rec)
    assert (to_np(rec) == c * g).all()


@pytest.mark.parametrize("M", [3, 4, 8])
def test_w32_random_faults(O, M):
    """Random-mask corruptions of random words of single streams: flags, d_hat
    (low 32 bits of the exact values) and the bitmap equal the oracle's, and
    every corrupted position is flagged (M l >= w: Props 2/4)."""
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    hi = ne.ne_dynamic_range(cfg)
    N = 4096 + 7
    c = gen(O, 7, 1, M, N, -hi, hi + 1)
    D = O.entangle(ocfg, c)
    rng = np.random.default_rng(M)
    pos = rng.choice(N, size=300, replace=False)
    D_f = D.copy()
    for p in pos:
        s = rng.integers(M)
        mask = int(rng.integers(1, 2 ** 32))
        D_f[s, p] = O.wrap(ocfg, int(D_f[s, p]) ^ mask)
    d_out = empty32(M, N)
    bm = torch.empty((N + 31) // 32, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_disentangle_check_w32(cfg, to_streams(D_f), 0, d_out, bm, diag)
    ref, flags, nf = O.disentangle_check(ocfg, D_f, 0)
    assert (to_np(d_out) == ref).all()
    assert (bitmap_to_flags(bm, N) == flags).all()
    d = ne.diag_read(diag)
    assert d["fault_positions"] == nf and nf == len(pos)
    assert d["first_fault"] == int(pos.min())


def test_w32_exhaustive_single_bit_injection(O):
    """All 3 x 64 x 32 single-bit flips of the C1 (w = 32) outputs in the first
    64 positions: exactly the injected position is flagged, and d_hat at it
    equals the oracle's for the same corrupted word."""
    M, N, W = 3, 4096, 64
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    c = gen(O, 0, 1, M, N, -2 ** 10, 2 ** 10)
    a = gen(O, 0, 2, M, N, -2 ** 10, 2 ** 10)
    D = O.op_add(ocfg, O.op_scale(ocfg, O.entangle(ocfg, c), 37), O.entangle(ocfg, a), 1)
    for r in (0, 2):
        T = M * W * 32
        fw = torch.empty(T, dtype=torch.int64, device="cuda")
        dh = torch.empty(T * M, dtype=torch.int32, device="cuda")
        ne.ne_inject_sweep_w32(cfg, to_streams(D[:, :W]), W, r, fw, dh)
        fw = fw.cpu().numpy().astype(np.uint64)
        dh = dh.cpu().numpy().reshape(T, M)
        for t in range(T):
            bit, p, s = t & 31, (t >> 5) % W, (t >> 5) // W
            assert fw[t] == np.uint64(1) << np.uint64(p), (r, s, p, bit)
            col = D[:, p].copy()
            col[s] = O.wrap(ocfg, int(col[s]) ^ (1 << bit))
            out, f = O.disentangle_one(ocfg, col, r)
            assert f == 1 and (dh[t] == out).all()


def test_w32_range_violation_names_first(O):
    M, N = 3, 5000
    cfg = ne.ne_config_for(M, 32)
    hi = ne.ne_dynamic_range(cfg)
    c = gen(O, 1, 1, M, N, -100, 100)
    c[2, 4000] = hi + 1
    c[1, 4001] = -hi - 1
    c[0, 17] = hi  # at the limit: admissible
    diag = ne.diag_new()
    ne.ne_entangle_w32(cfg, to_streams(c), empty32(M, N), diag)
    d = ne.diag_read(diag)
    assert d["range_violations"] == 2 and d["first_bad"] == 1 * N + 4001


@pytest.mark.parametrize("M,N,r", [(3, 4096, 0), (3, 4099, 1), (4, 1003, 3), (8, 515, 2), (5, 129, 4)])
def test_w32_scale_add_check_fused(O, M, N, r):
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    hi = ne.ne_dynamic_range(cfg)
    b = min(2 ** 10, hi // 40)
    c = gen(O, 15, 1, M, N, -b, b + 1)
    a = gen(O, 15, 2, M, N, -b, b + 1)
    E, A = O.entangle(ocfg, c), O.entangle(ocfg, a)
    for corrupt in (False, True):
        Ec = E.copy()
        if corrupt:
            Ec[(r + 1) % M, N // 2] = O.wrap(ocfg, int(Ec[(r + 1) % M, N // 2]) ^ (1 << 20))
        D = O.op_add(ocfg, O.op_scale(ocfg, Ec, 37), A, 1)
        ref, flags, nf = O.disentangle_check(ocfg, D, r)
        x = to_streams(Ec)
        d_out = empty32(M, N)
        bm = torch.full(((N + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        dg = ne.diag_new()
        ne.ne_op_scale_add_check_w32(cfg, x, 37, to_streams(A), r, d_out, bm, dg)
        assert (to_np(x) == D).all() and (to_np(d_out) == ref).all()
        assert (bitmap_to_flags(bm, N) == flags).all()
        assert ne.diag_read(dg)["fault_positions"] == nf and (nf == 1) == corrupt


@pytest.mark.parametrize("M,sets,N", [(3, 2, 4096), (3, 2, 4099), (4, 3, 1001)])
def test_w32_entangle_sets(O, M, sets, N):
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    hi = ne.ne_dynamic_range(cfg)
    c = np.concatenate([gen(O, 20 + s, 1, M, N, -hi, hi + 1) for s in range(sets)])
    eps = empty32(sets * M, N)
    diag = ne.diag_new()
    ne.ne_entangle_sets_w32(cfg, to_streams(c), sets, eps, diag)
    got = to_np(eps)
    for s in range(sets):
        assert (got[s * M:(s + 1) * M] == O.entangle(ocfg, c[s * M:(s + 1) * M])).all()
    assert ne.diag_read(diag)["range_violations"] == 0
    c[M + 2, 7] = hi + 1
    ne.ne_entangle_sets_w32(cfg, to_streams(c), sets, eps, diag)
    d = ne.diag_read(diag)
    assert d["range_violations"] == 1 and d["first_bad"] == (M + 2) * N + 7


# ------------------------------------------------------------------ C4 class at w = 32
@pytest.mark.parametrize("M,N", [(4, 4096 + 3), (4, 4096), (4, 65536 + 4), (3, 1000), (8, 515), (5, 129)])
def test_w32_entangle_aos(O, M, N):
    """x_aos[n*M + m] = eps_m[n] (Eq. 15 mod 2^32), range violations named."""
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    hi = ne.ne_dynamic_range(cfg)
    c = gen(O, 30, 1, M, N, -hi, hi + 1)
    c[:, 0], c[:, 1] = hi, -hi
    x = torch.empty(N * M, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_aos_w32(cfg, to_streams(c), x, diag)
    assert (x.view(N, M).cpu().numpy().T.astype(np.int64) == O.entangle(ocfg, c)).all()
    assert ne.diag_read(diag)["range_violations"] == 0
    c[M - 1, N - 1] = hi + 1
    ne.ne_entangle_aos_w32(cfg, to_streams(c), x, diag)
    d = ne.diag_read(diag)
    assert d["range_violations"] == 1 and d["first_bad"] == (M - 1) * N + N - 1


@pytest.mark.parametrize("M", [4, 3, 8, 5])
@pytest.mark.parametrize("gather", [True, False])
@pytest.mark.parametrize("vlen_eq_block", [True, False])
def test_w32_permute_inner_check(O, M, gather, vlen_eq_block):
    """Gather + blocked inner product + disentangle/check in w = 32 AoS
    containers: block sums (mod 2^32), d_hat, bitmap and diag equal the
    oracle's, and d_hat equals the plain inner products of the permuted c."""
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    hi = ne.ne_dynamic_range(cfg)
    B = 256
    vlen = B if vlen_eq_block else 96
    N = B * 37 + 100
    vb = 16
    cb = max(1, hi // (B * vb))          # every block sum inside the dynamic range
    c = gen(O, 31, 1, M, N, -cb, cb + 1)
    v = O.gen_uniform(31, 7, 0, -vb, vb + 1, vlen)
    perm = O.gen_perm(31, 6, N)
    E = O.entangle(ocfg, c)
    x = dev(E.T.copy(), torch.int32).reshape(-1)
    nb = (N + B - 1) // B
    d_out = [torch.empty(nb, dtype=torch.int32, device="cuda") for _ in range(M)]
    delta = [torch.empty(nb, dtype=torch.int32, device="cuda") for _ in range(M)]
    bm = torch.full(((nb + 31) // 32,), -1, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    r = 1 % M
    ne.ne_op_permute_inner_check_w32(cfg, x, dev(v, torch.int32), B, r, d_out,
                                     perm=dev(perm, torch.int32) if gather else None, delta_out=delta, bitmap=bm,
                                     diag=diag)
    p = perm if gather else np.arange(N)
    odelta = O.op_inner(ocfg, O.op_permute(E, p), v, B)
    assert (to_np(delta) == odelta).all()
    od, oflags, onf = O.disentangle_check(ocfg, odelta, r)
    assert (to_np(d_out) == od).all()
    assert (od == O.op_inner(O.config_for(M, 64), c[:, p], v, B)).all()
    assert (bitmap_to_flags(bm, nb) == oflags).all() and onf == 0
    assert ne.diag_read(diag)["fault_positions"] == 0


def test_w32_permute_inner_detects_storage_fault(O):
    """Single-stream faults in stored w = 32 words are flagged in their blocks;
    d_hat and flags equal the oracle's on the corrupted containers."""
    M, B = 4, 1024
    N = B * 64
    cfg, ocfg = ne.ne_config_for(M, 32), O.config_for(M, 32)
    c = gen(O, 32, 1, M, N, -64, 64)
    v = O.gen_uniform(32, 7, 0, -64, 64, B)
    perm = O.gen_perm(32, 6, N)
    x = O.entangle(ocfg, c).T.copy()
    hit = [(5, 2, 1 << 20), (40000 % N, 0, 1), (N - 1, 3, 1 << 31)]
    for pos, s, mask in hit:
        x[pos, s] = O.wrap(ocfg, int(x[pos, s]) ^ mask)
    nb = N // B
    d_out = [torch.empty(nb, dtype=torch.int32, device="cuda") for _ in range(M)]
    bm = torch.empty(nb // 32, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_op_permute_inner_check_w32(cfg, dev(x, torch.int32).reshape(-1), dev(v, torch.int32), B, 0, d_out,
                                     perm=dev(perm, torch.int32), bitmap=bm, diag=diag)
    inv = np.argsort(perm)
    blocks = sorted({int(inv[pos]) // B for pos, _, _ in hit})
    flags = bitmap_to_flags(bm, nb)
    assert list(np.flatnonzero(flags)) == blocks
    odelta = O.op_inner(ocfg, O.op_permute(np.ascontiguousarray(x.T), perm), v, B)
    od, oflags, _ = O.disentangle_check(ocfg, odelta, 0)
    assert (to_np(d_out) == od).all() and (oflags == flags).all()
    assert ne.diag_read(diag)["fault_positions"] == len(blocks)
