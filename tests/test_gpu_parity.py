"""GPU parity: every stage of the hot path through the C ABI (libne.so, sm_100a)
against the CPU oracle on the same seeded inputs, bit-exact (all work is
integer).  Sizes span several tiles plus ragged tails; edge cases cover empty
inputs, M = 3..32, every excluded stream, maximal values and faults."""
import numpy as np
import pytest
import torch

import paper_1604_04740_b200 as ne
from _gpu import bitmap_to_flags, dev, empty_streams, to_np, to_streams

pytestmark = pytest.mark.gpu

MS = [3, 4, 5, 8, 11, 16, 32]


@pytest.fixture(scope="module", autouse=True)
def _lib():
    ne.build()
    ne.lib()
    assert torch.cuda.is_available()


def gen(O, seed, tag, M, N, lo, hi):
    return np.stack([O.gen_uniform(seed, tag, m, lo, hi, N) for m in range(M)])


# ------------------------------------------------------------------ inputs
@pytest.mark.parametrize("N", [1, 5, 4096, 100003])
def test_generator_parity(O, N):
    out = torch.empty(N, dtype=torch.int32, device="cuda")
    for (seed, tag, st, lo, hi) in [(0, 1, 2, -1024, 1024), (3, 4, 0, -2 ** 31, 2 ** 31 - 1), (9, 7, 1, 0, 1)]:
        ne.ne_gen_uniform_i32(seed, tag, st, lo, hi, out)
        assert (out.cpu().numpy() == O.gen_uniform(seed, tag, st, lo, hi, N)).all()
    ne.ne_gen_perm_i32(5, 6, out)
    assert (out.cpu().numpy() == O.gen_perm(5, 6, N)).all()


# ------------------------------------------------------------------ a1 / a2
@pytest.mark.parametrize("M", MS)
@pytest.mark.parametrize("N", [1, 3, 4, 1029, 65536 + 7])
def test_entangle_soa(O, M, N):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    hi = O.dynamic_range(ocfg)
    lim = min(hi, 2 ** 31 - 1)
    c = gen(O, M, 1, M, N, -lim, lim + 1)
    eps = empty_streams(M, N)
    diag = ne.diag_new()
    ne.ne_entangle(cfg, to_streams(c), eps, diag)
    assert (to_np(eps) == O.entangle(ocfg, c)).all()
    d = ne.diag_read(diag)
    assert d["range_violations"] == O.range_check(c, hi)[0]


def test_entangle_range_violation_names_first(O):
    """a0: values the output format cannot hold are counted and the first is
    named m*N + n.  With w = 64 every int32 input is inside Eq. 13's
    range, so the limb format (L = 1 digit: [-128, 127]) exercises the path."""
    cfg, ocfg = ne.ne_config_for(3), O.config_for(3, 64)
    N = 1008
    c = np.zeros((3, N), dtype=np.int64)
    c[1, 17] = 5000
    c[2, 3] = -4000
    planes = torch.empty(3 * N, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, to_streams(c), 1, planes, diag)
    d = ne.diag_read(diag)
    eps = O.entangle(ocfg, c)
    bad = np.argwhere((eps > 127) | (eps < -128))
    assert d["range_violations"] == len(bad) > 0
    assert d["first_bad"] == min(m * N + n for m, n in bad)


@pytest.mark.parametrize("M", [3, 4, 8, 5])
@pytest.mark.parametrize("N", [1, 7, 4096 + 5])
def test_entangle_aos(O, M, N):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 11, 1, M, N, -2 ** 12, 2 ** 12)
    aos = torch.empty(N * M, dtype=torch.int64, device="cuda")
    ne.ne_entangle_aos(cfg, to_streams(c), aos)
    assert (aos.cpu().numpy().reshape(N, M).T == O.entangle(ocfg, c)).all()


@pytest.mark.parametrize("M,L,B", [(3, 4, 64), (8, 2, 32), (4, 4, 1000), (3, 3, 1), (3, 1, 0), (5, 3, 1)])
def test_entangle_limbs(O, M, L, B):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    N = 4096 + 16
    c = gen(O, 2, 4, M, N, -B, B + 1)
    planes = torch.empty(M * L * N, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, to_streams(c), L, planes, diag)
    p = planes.cpu().numpy().astype(np.int64).reshape(M, L, N)
    recon = sum(p[:, i, :] * (256 ** i) for i in range(L))
    assert (recon == O.entangle(ocfg, c)).all()
    assert p.min() >= -128 and p.max() <= 127
    assert ne.diag_read(diag)["range_violations"] == 0


@pytest.mark.parametrize("M", [3, 8])
def test_entangle_stream_and_shared(O, M):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    N = 3001
    c = gen(O, 4, 1, M, N, -32, 32)
    ref = O.entangle(ocfg, c)
    cs = to_streams(c)
    for m in range(M):
        out = torch.empty(N, dtype=torch.int64, device="cuda")
        ne.ne_entangle_stream(cfg, m, cs[m], cs[(m - 1) % M], out)
        assert (out.cpu().numpy() == ref[m]).all()
    g = O.gen_uniform(1, 2, 0, -1000, 1000, N)
    ge = torch.empty(N, dtype=torch.int64, device="cuda")
    ne.ne_entangle_shared(cfg, dev(g, torch.int32), ge)
    assert (ge.cpu().numpy() == O.entangle_shared(ocfg, g)).all()


# ------------------------------------------------------------------ a4 / a5 / a6
@pytest.mark.parametrize("M", MS)
@pytest.mark.parametrize("N", [1, 2, 63, 64, 65, 4096 + 33])
def test_disentangle_check_clean_and_faulty(O, M, N):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    hi = O.dynamic_range(ocfg)
    rng = np.random.default_rng(M * 1000 + N)
    c = rng.integers(-hi, hi + 1, size=(M, N))
    c[:, 0] = hi
    delta = O.entangle(ocfg, c)
    # corrupt ~1/8 of positions in one random stream with a random 64-bit mask
    bad = rng.random(N) < 0.125
    for n in np.flatnonzero(bad):
        s = rng.integers(0, M)
        delta[s, n] ^= np.int64(rng.integers(1, 2 ** 63))
    for r in sorted({0, M - 1, int(rng.integers(0, M))}):
        d_out = empty_streams(M, N)
        bm = torch.full(((N + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        diag = ne.diag_new()
        ne.ne_disentangle_check(cfg, to_streams(delta, torch.int64), r, d_out, bm, diag)
        od, oflags, onf = O.disentangle_check(ocfg, delta, r)
        assert (to_np(d_out) == od).all()
        assert (bitmap_to_flags(bm, N) == oflags).all()
        d = ne.diag_read(diag)
        assert d["fault_positions"] == onf == int(bad.sum())  # every single-stream fault caught
        assert d["first_fault"] == (int(np.flatnonzero(oflags)[0]) if onf else None)


@pytest.mark.parametrize("M", MS)
def test_recover_every_stream(O, M):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    hi = O.dynamic_range(ocfg)
    N = 5003
    rng = np.random.default_rng(M)
    c = rng.integers(-hi, hi + 1, size=(M, N))
    delta = O.entangle(ocfg, c)
    ds = to_streams(delta, torch.int64)
    for r in range(M):
        part = [None if m == r else ds[m] for m in range(M)]
        d_out = empty_streams(M, N)
        ne.ne_recover(cfg, part, r, d_out)
        assert (to_np(d_out) == c).all()
    with pytest.raises(ne.NeError):
        ne.ne_recover(cfg, [None, None] + ds[2:], 0, empty_streams(M, N))


def test_empty_and_bad_args():
    cfg = ne.ne_config_for(3)
    z = empty_streams(3, 0)
    ne.ne_disentangle_check(cfg, z, 0, empty_streams(3, 0))
    with pytest.raises(ne.NeError):
        ne.ne_disentangle_check(cfg, empty_streams(3, 8), 3, empty_streams(3, 8))
    base = torch.empty(9, dtype=torch.int64, device="cuda")
    with pytest.raises(ne.NeError):  # misaligned stream pointer
        ne.ne_op_scale(cfg, [base[1:5], base[1:5], base[1:5]], 2)


# ------------------------------------------------------------------ C1 (BASELINE configs[0])
def c1_pipeline_oracle(O, c, a, s=37):
    ocfg = O.config_for(3, 64)
    eps = O.entangle(ocfg, c)
    delta = O.op_add(ocfg, O.op_scale(ocfg, eps, s), O.entangle(ocfg, a), 1)
    return ocfg, delta


def test_c1_full_chain(O):
    """C1: M=3, N=4096, c,a ~ U[-2^10, 2^10) (seed 0), eps = E c, alpha = E a,
    delta = 37 eps + alpha, disentangle + check (r = 0), recovery of every r."""
    M, N = 3, 4096
    cfg = ne.ne_config_for(M)
    c_dev = [torch.empty(N, dtype=torch.int32, device="cuda") for _ in range(M)]
    a_dev = [torch.empty(N, dtype=torch.int32, device="cuda") for _ in range(M)]
    for m in range(M):
        ne.ne_gen_uniform_i32(0, 1, m, -1024, 1024, c_dev[m])
        ne.ne_gen_uniform_i32(0, 2, m, -1024, 1024, a_dev[m])
    c = gen(O, 0, 1, M, N, -1024, 1024)
    a = gen(O, 0, 2, M, N, -1024, 1024)
    assert (to_np(c_dev) == c).all() and (to_np(a_dev) == a).all()
    eps, alpha = empty_streams(M, N), empty_streams(M, N)
    diag = ne.diag_new()
    ne.ne_entangle(cfg, c_dev, eps, diag)
    ne.ne_entangle(cfg, a_dev, alpha, diag)
    ne.ne_op_scale(cfg, eps, 37)
    ne.ne_op_add(cfg, eps, alpha, 1)
    ocfg, delta = c1_pipeline_oracle(O, c, a)
    assert (to_np(eps) == delta).all()
    d_out = empty_streams(M, N)
    bm = torch.empty(N // 32, dtype=torch.int32, device="cuda")
    ne.ne_disentangle_check(cfg, eps, 0, d_out, bm, diag)
    od, oflags, onf = O.disentangle_check(ocfg, delta, 0)
    assert (to_np(d_out) == od).all() and (od == 37 * c + a).all()
    assert onf == 0 and (bitmap_to_flags(bm, N) == 0).all()
    dd = ne.diag_read(diag)
    assert dd["range_violations"] == 0 and dd["fault_positions"] == 0
    for r in range(M):
        part = [None if m == r else eps[m] for m in range(M)]
        rec = empty_streams(M, N)
        ne.ne_recover(cfg, part, r, rec)
        assert (to_np(rec) == od).all()


def test_c1_exhaustive_single_bit_injection(O):
    """C1 a7: all 3 x 64 x 64 = 12 288 single-bit flips of the first 64 outputs;
    each must flag exactly its own position, and (flag, d_hat) must equal the
    oracle's for the same corrupted tuple."""
    M, N, W = 3, 4096, 64
    cfg = ne.ne_config_for(M)
    c = gen(O, 0, 1, M, N, -1024, 1024)
    a = gen(O, 0, 2, M, N, -1024, 1024)
    ocfg, delta = c1_pipeline_oracle(O, c, a)
    T = M * W * 64
    fw = torch.empty(T, dtype=torch.int64, device="cuda")
    dh = torch.empty(T * M, dtype=torch.int64, device="cuda")
    ne.ne_inject_sweep(cfg, to_streams(delta, torch.int64), W, 0, fw, dh)
    fw = fw.cpu().numpy().view(np.uint64)
    dh = dh.cpu().numpy().reshape(T, M)
    for t in range(T):
        s, n, bit = t // (W * 64), (t // 64) % W, t % 64
        col = delta[:, n].copy()
        col[s] = np.int64(np.uint64(col[s]) ^ np.uint64(1 << bit))
        od, of = O.disentangle_one(ocfg, col, 0)
        assert of == 1
        assert int(fw[t]) == (1 << n), (s, n, bit)
        assert (dh[t] == od).all(), (s, n, bit)


# ------------------------------------------------------------------ a3 ops
@pytest.mark.parametrize("M", [3, 4, 8, 5])
@pytest.mark.parametrize("N", [1, 17, 4096 + 3])
def test_scale_add_elementwise(O, M, N):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    rng = np.random.default_rng(N + M)
    x = rng.integers(-2 ** 40, 2 ** 40, size=(M, N))
    g = rng.integers(-2 ** 31, 2 ** 31, size=N)
    xs = to_streams(x, torch.int64)
    ne.ne_op_scale(cfg, xs, -12345)
    assert (to_np(xs) == O.op_scale(ocfg, x, -12345)).all()
    ne.ne_op_scale(cfg, xs, 0, dev(g, torch.int32))
    ref = O.op_scale(ocfg, O.op_scale(ocfg, x, -12345), g=g)
    assert (to_np(xs) == ref).all()
    a = rng.integers(-2 ** 62, 2 ** 62, size=(M, N))
    ne.ne_op_add(cfg, xs, to_streams(a, torch.int64), -1)
    assert (to_np(xs) == O.op_add(ocfg, ref, a, -1)).all()
    ref2 = O.op_add(ocfg, ref, a, -1)
    ne.ne_op_scale_add(cfg, xs, -7, to_streams(a, torch.int64), 1)       # fused scale + add
    ref2 = O.op_add(ocfg, O.op_scale(ocfg, ref2, -7), a, 1)
    assert (to_np(xs) == ref2).all()
    gg = rng.integers(-2 ** 31, 2 ** 31, size=N)
    ne.ne_op_scale_add(cfg, xs, 1, to_streams(a, torch.int64), -1, dev(gg, torch.int32))
    assert (to_np(xs) == O.op_add(ocfg, O.op_scale(ocfg, ref2, 1, gg), a, -1)).all()


@pytest.mark.parametrize("N,T", [(65536, 64), (1000, 64), (777, 1), (50, 300), (4099, 2500)])
@pytest.mark.parametrize("correlate", [False, True])
def test_conv(O, N, T, correlate):
    M = 3
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 1, 1, M, N, -128, 128)
    g = O.gen_uniform(1, 3, 0, -128, 128, T)
    eps = O.entangle(ocfg, c)
    out = empty_streams(M, N)
    ne.ne_op_conv(cfg, to_streams(eps, torch.int64), dev(g, torch.int32), out, correlate)
    assert (to_np(out) == O.op_conv(ocfg, eps, g, correlate)).all()


def test_conv_int64_path(O):
    """Windows that do not fit int32 take the full 64-bit MAC path."""
    cfg, ocfg = ne.ne_config_for(3), O.config_for(3, 64)
    rng = np.random.default_rng(5)
    x = rng.integers(-2 ** 62, 2 ** 62, size=(3, 3000))
    g = rng.integers(-2 ** 31, 2 ** 31, size=70)
    out = empty_streams(3, 3000)
    ne.ne_op_conv(cfg, to_streams(x, torch.int64), dev(g, torch.int32), out)
    assert (to_np(out) == O.op_conv(ocfg, x, g)).all()


def test_c2_conv_full_pipeline(O):
    """C2: M=3, N=65536, c ~ U[-128,128) seed 1, 64 taps ~ U[-128,128):
    entangle -> circular conv -> disentangle + check == plain circular conv."""
    M, N, T = 3, 65536, 64
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 1, 1, M, N, -128, 128)
    g = O.gen_uniform(1, 3, 0, -128, 128, T)
    eps = empty_streams(M, N)
    ne.ne_entangle(cfg, to_streams(c), eps)
    out = empty_streams(M, N)
    ne.ne_op_conv(cfg, eps, dev(g, torch.int32), out)
    d_out = empty_streams(M, N)
    diag = ne.diag_new()
    ne.ne_disentangle_check(cfg, out, 0, d_out, None, diag)
    assert (to_np(d_out) == O.op_conv(O.config_for(M, 64), c, g)).all()
    assert ne.diag_read(diag)["fault_positions"] == 0


@pytest.mark.parametrize("M", [3, 4, 8, 6])
@pytest.mark.parametrize("N,block,vlen", [(1024 * 40, 1024, 1024), (5000, 1024, 1024), (1000, 16, 16),
                                          (3333, 100, 3333), (64, 1024, 1024)])
def test_inner(O, M, N, block, vlen):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    rng = np.random.default_rng(N)
    x = rng.integers(-2 ** 40, 2 ** 40, size=(M, N))
    v = rng.integers(-2 ** 12, 2 ** 12, size=vlen)
    nb = (N + block - 1) // block
    out = empty_streams(M, nb)
    ne.ne_op_inner(cfg, to_streams(x, torch.int64), dev(v, torch.int32), block, out)
    assert (to_np(out) == O.op_inner(ocfg, x, v, block)).all()


@pytest.mark.parametrize("M", [3, 4, 8, 5])
@pytest.mark.parametrize("aos", [True, False])
@pytest.mark.parametrize("gather", [True, False])
def test_permute_inner_check(O, M, aos, gather):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    N, B = 1024 * 37 + 500, 1024
    c = gen(O, 3, 1, M, N, -2 ** 12, 2 ** 12)
    perm = O.gen_perm(3, 6, N)
    v = O.gen_uniform(3, 7, 0, -2 ** 12, 2 ** 12, B)
    eps = O.entangle(ocfg, c)
    # inject single-stream faults into a few stored eps values -> those blocks flag
    nb = (N + B - 1) // B
    xs = to_streams(eps, torch.int64)
    x_aos = dev(eps.T.copy(), torch.int64).reshape(-1)
    d_out, delta = empty_streams(M, nb), empty_streams(M, nb)
    bm = torch.empty((nb + 31) // 32, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_op_permute_inner_check(cfg, dev(v, torch.int32), B, 1 % M, d_out,
                                 x=None if aos else xs, x_aos=x_aos if aos else None,
                                 perm=dev(perm, torch.int32) if gather else None, n=N,
                                 delta_out=delta, bitmap=bm, diag=diag)
    p = perm if gather else np.arange(N)
    odelta = O.op_inner(ocfg, O.op_permute(eps, p), v, B)
    assert (to_np(delta) == odelta).all()
    od, oflags, onf = O.disentangle_check(ocfg, odelta, 1 % M)
    assert (to_np(d_out) == od).all()
    assert (od == O.op_inner(O.config_for(M, 64), c[:, p], v, B)).all()
    assert (bitmap_to_flags(bm, nb) == oflags).all() and onf == 0
    assert ne.diag_read(diag)["fault_positions"] == 0


@pytest.mark.parametrize("M,N,B,vlen", [(4, 1024 * 37 + 500, 1024, 1024), (3, 100003, 100, 100), (8, 65536, 1024, 1024),
                                        (5, 4099, 7, 3), (4, 1 << 20, 1024, 1024), (4, 1, 1024, 1024),
                                        (4, 70000, 4096, 4096), (4, 300001, 2048, 2048), (3, (1 << 19) + 77, 512, 300),
                                        (8, 200003, 256, 256), (5, 1 << 21, 1024, 1000),
                                        (4, 100000, 3000, 3000)])
def test_permute_inner_bucketed(O, M, N, B, vlen):
    """The bucketed scatter-reduce form of the C4 op (ne_op_permute_inner_check_
    bucketed): delta, d_hat, bitmap and diag equal to the oracle's gather +
    blocked inner product + disentangle/check and bit-identical to the
    gather kernel — ragged n (last window and last block partial), block !=
    vlen, M = 3..8, windows from 16 up (n = 2^21), a block above 2048 in
    the shared-sum plan (3000: its 64-bit path), both plans (owned runs for power-of-two
    blocks 256-4096 — one, two and four blocks per scatter chunk, the
    16-byte and the scalar run-index stores — shared-memory sums for
    blocks 7, 100 and 3000), run twice on the same workspace."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 5, 1, M, N, -2 ** 12, 2 ** 12)
    perm = O.gen_perm(5, 6, N)
    v = O.gen_uniform(5, 7, 0, -2 ** 12, 2 ** 12, vlen)
    eps = O.entangle(ocfg, c)
    x_aos = dev(eps.T.copy(), torch.int64).reshape(-1)
    nb = (N + B - 1) // B
    ws = torch.empty(ne.ne_permute_inner_workspace(cfg, N, B), dtype=torch.uint8, device="cuda")
    p = perm
    idx = np.arange(N)
    odelta = np.zeros((M, nb), dtype=np.int64)
    prod = (eps[:, p].astype(np.int64) * v[idx % vlen].astype(np.int64))   # |eps v| < 2^29 2^12: exact
    for m in range(M):
        odelta[m] = np.add.reduceat(prod[m], np.arange(0, N, B)) if N > 0 else 0
    if vlen == B:
        assert (odelta == O.op_inner(ocfg, O.op_permute(eps, p), v, B)).all()   # the oracle's own definition
    od, oflags, onf = O.disentangle_check(ocfg, odelta, 2 % M)
    for _ in range(2):
        delta, d_out = empty_streams(M, nb), empty_streams(M, nb)
        bm = torch.full(((nb + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        diag = ne.diag_new()
        ne.ne_op_permute_inner_check_bucketed(cfg, x_aos, dev(perm, torch.int32), dev(v, torch.int32), B, 2 % M,
                                              delta, d_out, ws, bm, diag)
        torch.cuda.synchronize()
        assert (to_np(delta) == odelta).all()
        assert (to_np(d_out) == od).all()
        assert (bitmap_to_flags(bm, nb) == oflags).all() and onf == 0
        dd = ne.diag_read(diag)
        assert dd["fault_positions"] == 0 and dd["range_violations"] == 0
    if vlen == B:
        d2 = empty_streams(M, nb)
        g = empty_streams(M, nb)
        ne.ne_op_permute_inner_check(cfg, dev(v, torch.int32), B, 2 % M, d2, x_aos=x_aos,
                                     perm=dev(perm, torch.int32), n=N, delta_out=g)
        assert all(torch.equal(a, b) for a, b in zip(g, delta)) and all(torch.equal(a, b) for a, b in zip(d2, d_out))


@pytest.mark.parametrize("kind", ["identity", "reverse", "local"])
def test_permute_inner_bucketed_skewed_perm(O, kind):
    """Permutations far from random fill some cells past their capacity (a
    random permutation's mean + 8 sigma): those pairs take the overflow list
    (global 64-bit reductions after the reduce pass) — identity, reversal and
    a shuffle inside 4096-position windows, against the oracle."""
    M, N, B = 4, 1 << 18, 1024
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 8, 1, M, N, -2 ** 12, 2 ** 12)
    v = O.gen_uniform(8, 7, 0, -2 ** 12, 2 ** 12, B)
    if kind == "identity":
        perm = np.arange(N, dtype=np.int32)
    elif kind == "reverse":
        perm = np.arange(N - 1, -1, -1, dtype=np.int32)
    else:
        perm = np.concatenate([w0 + O.gen_perm(8, 9 + w0 // 4096, 4096) for w0 in range(0, N, 4096)]).astype(np.int32)
    eps = O.entangle(ocfg, c)
    nb = N // B
    odelta = O.op_inner(ocfg, O.op_permute(eps, perm), v, B)
    od, _, _ = O.disentangle_check(ocfg, odelta, 0)
    ws = torch.empty(ne.ne_permute_inner_workspace(cfg, N, B), dtype=torch.uint8, device="cuda")
    delta, d_out = empty_streams(M, nb), empty_streams(M, nb)
    diag = ne.diag_new()
    ne.ne_op_permute_inner_check_bucketed(cfg, dev(eps.T.copy(), torch.int64).reshape(-1), dev(perm, torch.int32),
                                          dev(v, torch.int32), B, 0, delta, d_out, ws, None, diag)
    assert (to_np(delta) == odelta).all() and (to_np(d_out) == od).all()
    assert ne.diag_read(diag)["fault_positions"] == 0


def test_permute_inner_bucketed_bad_perm_and_fault(O):
    """perm entries outside [0, n) are counted (first named) and skipped; a
    stored-eps fault in one stream flags exactly its block, as the gather
    path does."""
    M, N, B = 4, 1024 * 64, 1024
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 6, 1, M, N, -2 ** 12, 2 ** 12)
    perm = O.gen_perm(6, 6, N)
    v = O.gen_uniform(6, 7, 0, -2 ** 12, 2 ** 12, B)
    eps = O.entangle(ocfg, c)
    xa = eps.T.copy()
    xa[perm[5000], 1] = np.int64(np.uint64(xa[perm[5000], 1]) ^ np.uint64(1 << 33))   # position 5000's source
    x_aos = dev(xa, torch.int64).reshape(-1)
    nb = N // B
    ws = torch.empty(ne.ne_permute_inner_workspace(cfg, N, B), dtype=torch.uint8, device="cuda")
    delta, d_out = empty_streams(M, nb), empty_streams(M, nb)
    bm = torch.empty(nb // 32, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_op_permute_inner_check_bucketed(cfg, x_aos, dev(perm, torch.int32), dev(v, torch.int32), B, 0, delta,
                                          d_out, ws, bm, diag)
    flags = bitmap_to_flags(bm, nb)
    assert flags.sum() == 1 and flags[5000 // B]
    assert ne.diag_read(diag)["fault_positions"] == 1
    bad = perm.copy()
    bad[[17, 40000]] = [-3, N + 5]
    diag = ne.diag_new()
    ne.ne_op_permute_inner_check_bucketed(cfg, dev(eps.T.copy(), torch.int64).reshape(-1), dev(bad, torch.int32),
                                          dev(v, torch.int32), B, 0, delta, d_out, ws, None, diag)
    dd = ne.diag_read(diag)
    assert dd["range_violations"] == 2 and dd["first_bad"] == 17


def test_permute_inner_detects_storage_fault(O):
    """A fault in one stored eps word (one stream) is caught in its block."""
    M, N, B = 4, 1024 * 64, 1024
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 3, 1, M, N, -2 ** 12, 2 ** 12)
    perm = O.gen_perm(3, 6, N)
    v = O.gen_uniform(3, 7, 0, -2 ** 12, 2 ** 12, B)
    eps = O.entangle(ocfg, c)
    x_aos = eps.T.copy()
    hit = [(5, 2, 1 << 40), (70000 % N, 0, 1), (N - 1, 3, 1 << 63)]
    for pos, s, mask in hit:
        x_aos[pos, s] = np.int64(np.uint64(x_aos[pos, s]) ^ np.uint64(mask))
    nb = N // B
    d_out = empty_streams(M, nb)
    bm = torch.empty(nb // 32, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_op_permute_inner_check(cfg, dev(v, torch.int32), B, 0, d_out, x_aos=dev(x_aos, torch.int64).reshape(-1),
                                 perm=dev(perm, torch.int32), n=N, bitmap=bm, diag=diag)
    inv = np.argsort(perm)
    blocks = sorted({int(inv[pos]) // B for pos, _, _ in hit})
    flags = bitmap_to_flags(bm, nb)
    assert list(np.flatnonzero(flags)) == blocks
    odelta = O.op_inner(ocfg, O.op_permute(np.ascontiguousarray(x_aos.T), perm), v, B)
    od, oflags, _ = O.disentangle_check(ocfg, odelta, 0)
    assert (to_np(d_out) == od).all() and (oflags == flags).all()
    assert ne.diag_read(diag)["fault_positions"] == len(blocks)


@pytest.mark.parametrize("M", [3, 8])
def test_permute_outer(O, M):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    N = 10007
    rng = np.random.default_rng(2)
    x = rng.integers(-2 ** 40, 2 ** 40, size=(M, N))
    perm = O.gen_perm(8, 6, N)
    out = empty_streams(M, N)
    ne.ne_op_permute(cfg, to_streams(x, torch.int64), dev(perm, torch.int32), out)
    assert (to_np(out) == O.op_permute(x, perm)).all()
    for n1, n2 in [(37, 64), (100, 33), (1, 1)]:
        h = rng.integers(-2 ** 31, 2 ** 31, size=n2)
        xs = x[:, :n1].copy()
        o = empty_streams(M, n1 * n2)
        ne.ne_op_outer(cfg, to_streams(xs, torch.int64), dev(h, torch.int32), o)
        assert (to_np(o) == O.op_outer(ocfg, xs, h).reshape(M, -1)).all()


# ------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("rows,cols,K", [(64, 64, 16), (100, 37, 129), (256, 128, 384), (1, 1, 1)])
def test_gemm_imad64(O, rows, cols, K):
    M = 3
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    A = np.stack([O.gen_uniform(2, 4, m, -64, 64, rows * K) for m in range(M)])
    B = O.gen_uniform(2, 5, 0, -64, 64, K * cols)
    E = O.entangle(ocfg, A)
    out = empty_streams(M, rows * cols)
    ne.ne_op_gemm(cfg, to_streams(E, torch.int64), dev(B, torch.int32), rows, cols, K, out, algo=ne.NE_GEMM_IMAD64)
    ref = O.op_gemm(ocfg, E.reshape(M, rows, K), B.reshape(K, cols)).reshape(M, -1)
    assert (to_np(out) == ref).all()


@pytest.mark.parametrize("rows,cols,K", [(128, 128, 16), (256, 384, 4096), (100, 37, 129)])
def test_gemm_imad32w(O, rows, cols, K):
    """The CUDA-core comparison point with one IMAD.WIDE per MAC (every
    entangled entry fits int32, C3's operand): equal to the oracle; a shape
    that is not tile-aligned runs the 64-bit form, same result."""
    M = 3
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    A = np.stack([O.gen_uniform(3, 4, m, -64, 64, rows * K) for m in range(M)])
    B = O.gen_uniform(3, 5, 0, -2 ** 31, 2 ** 31 - 1, K * cols)
    E = O.entangle(ocfg, A)
    out = empty_streams(M, rows * cols)
    diag = ne.diag_new()
    ne.ne_op_gemm(cfg, to_streams(E, torch.int64), dev(B, torch.int32), rows, cols, K, out,
                  algo=ne.NE_GEMM_IMAD32W, diag=diag)
    assert ne.diag_read(diag)["range_violations"] == 0
    ref = O.op_gemm(ocfg, E.reshape(M, rows, K), B.reshape(K, cols)).reshape(M, -1)
    assert (to_np(out) == ref).all()


def test_gemm_imad32w_range_violation(O):
    """An entangled entry outside int32 is named in diag (the 64-bit form is
    the one for such operands)."""
    M, rows, cols, K = 3, 128, 128, 32
    cfg = ne.ne_config_for(M)
    E = np.zeros((M, rows * K), dtype=np.int64)
    E[1, 5 * K + 7] = 2 ** 31
    E[2, 3] = -2 ** 31 - 1
    out = empty_streams(M, rows * cols)
    diag = ne.diag_new()
    ne.ne_op_gemm(cfg, to_streams(E, torch.int64), torch.ones(K * cols, dtype=torch.int32, device="cuda"), rows,
                  cols, K, out, algo=ne.NE_GEMM_IMAD32W, diag=diag)
    d = ne.diag_read(diag)
    assert d["range_violations"] == 2 and d["first_bad"] == 1 * rows * K + 5 * K + 7


@pytest.mark.parametrize("M,L,bound,rows,cols,K", [
    (3, 4, 64, 128, 128, 128), (3, 4, 64, 256, 384, 512), (8, 2, 32, 128, 256, 256),
    (4, 4, 1000, 128, 128, 1024), (3, 3, 1, 128, 128, 256), (3, 1, 0, 128, 256, 128), (8, 2, 32, 256, 128, 128)])
def test_gemm_tc_i8(O, M, L, bound, rows, cols, K):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    assert ne.ne_gemm_limbs_for(cfg, bound) <= L
    A = np.stack([O.gen_uniform(2, 4, m, -bound, bound + 1, rows * K) for m in range(M)])
    B = O.gen_uniform(2, 5, 0, -64, 64, K * cols)
    E = O.entangle(ocfg, A)
    ref = O.op_gemm(ocfg, E.reshape(M, rows, K), B.reshape(K, cols)).reshape(M, -1)
    # int64 entangled operand path (split in the op)
    out = empty_streams(M, rows * cols)
    ws = torch.empty(ne.ne_gemm_workspace(cfg, rows, cols, K, L), dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_op_gemm(cfg, to_streams(E, torch.int64), dev(B, torch.int32), rows, cols, K, out,
                  algo=ne.NE_GEMM_TC_I8, L=L, ws=ws, diag=diag)
    torch.cuda.synchronize()
    assert ne.diag_read(diag)["range_violations"] == 0
    assert (to_np(out) == ref).all()
    # limb-plane path fed straight from the entangle kernel
    planes = torch.empty(M * L * rows * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes)
    Bt = torch.empty(cols * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, cols, Bt)
    out2 = empty_streams(M, rows * cols)
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, rows, cols, K, out2)
    assert (to_np(out2) == ref).all()
    d_out = empty_streams(M, rows * cols)
    ne.ne_disentangle_check(cfg, out2, 0, d_out, None, diag)
    plain = (A.reshape(M, rows, K) @ B.reshape(K, cols)).reshape(M, -1)
    assert (to_np(d_out) == plain).all()
    assert ne.diag_read(diag)["fault_positions"] == 0


@pytest.mark.parametrize("M,bound,R,Cc,K", [(3, 127, 256, 512, 4096), (4, 127, 256, 256, 4096),
                                            (8, 32, 256, 256, 8192), (3, 64, 512, 256, 6144)])
def test_gemm_pair_limb_major(O, M, bound, R, Cc, K):
    """Two-digit GEMMs with 4096 <= K <= 8192 run on the CTA-pair kernel with
    limb-major passes (k_gemm_pair.cu: 256 x 256 pair tiles, cta_group::2, the
    limb-1 accumulators held in registers while limb 0 drains): bit-exact
    against the oracle, in full, for every pair plan base (l = 22, 16, 8) and
    both passes, and the digits of every stream (one tile per pair at these
    sizes; the multi-tile path is test_gemm_pair_multi_tile_full)."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, bound)
    assert L == 2 and b == cfg.l
    assert ne.ne_gemm_kernel_for(cfg, L, b, R, Cc, K) == "pair"
    A = gen(O, 80, 4, M, R * K, -bound, bound + 1)
    A[:, 0], A[:, -1] = bound, -bound
    B = O.gen_uniform(80, 5, 0, -128, 128, K * Cc)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    out = empty_streams(M, R * Cc)
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, limb_bits=b)
    ref = O.op_gemm(ocfg, O.entangle(ocfg, A).reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    assert (to_np(out) == ref).all()


def test_gemm_pair_multi_tile(O):
    """The pair kernel's multi-tile path (several pair tiles per SM pair: the
    limb-1 hold in registers, the early tmem_empty release, barrier phase
    flips across tiles), with the persistent grid capped (ne_gemm_trace with
    no buffer) at 1 and 2 pairs so a pair walks 6-12 tiles of 3 streams:
    rows in every 32-lane group of both 128-row halves vs the oracle, and the
    whole output by a Freivalds identity (x in [-2, 2): |E (B x)| < 2^62)."""
    M, R, Cc, K = 3, 256, 1024, 4096
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, 127)
    assert ne.ne_gemm_kernel_for(cfg, L, b, R, Cc, K) == "pair"
    A = gen(O, 82, 4, M, R * K, -127, 128)
    B = O.gen_uniform(82, 5, 0, -128, 128, K * Cc)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    E = O.entangle(ocfg, A).reshape(M, R, K)
    rows = _band_rows(R, 128, seed=5)
    ref = O.op_gemm(ocfg, E[:, rows], B.reshape(K, Cc))
    x = np.random.default_rng(2).integers(-2, 2, size=Cc)
    bx = B.reshape(K, Cc) @ x
    for cap in (1, 2):
        out = empty_streams(M, R * Cc)
        ne.ne_gemm_trace(None, cap)
        try:
            ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, limb_bits=b)
            torch.cuda.synchronize()
        finally:
            ne.ne_gemm_trace(None, 0)
        got = np.stack([out[m].view(R, Cc)[torch.from_numpy(rows).cuda()].cpu().numpy() for m in range(M)])
        assert (got == ref).all(), cap
        for m in range(M):
            assert (out[m].cpu().numpy().reshape(R, Cc) @ x == E[m] @ bx).all(), (cap, m)


@pytest.mark.parametrize("cap", [0, 4, 8])
def test_gemm_pair_half_tiles(O, cap):
    """The pair kernel's 256 x 128 half tiles (N = 128 MMAs, a quarter of the
    B columns per CTA through the half-box tensor map, 4 epilogue chunks per
    warp): every tile halved (debug hook), every tile whole, and the
    automatic schedule (a last partial wave halved), with the full grid
    (automatic: all 18 tiles halved) and with 4 or 8 pairs (automatic: 16
    whole tiles, then 4 halves — halves after whole tiles on one pair):
    bit-identical, and equal to the oracle on rows in every lane group plus
    a Freivalds identity over the whole output."""
    M, R, Cc, K = 3, 512, 768, 4096     # 18 pair tiles
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, 127)
    assert ne.ne_gemm_kernel_for(cfg, L, b, R, Cc, K) == "pair"
    A = gen(O, 87, 4, M, R * K, -127, 128)
    A[:, 0], A[:, -1] = 127, -127
    B = O.gen_uniform(87, 5, 0, -128, 128, K * Cc)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    outs = {}
    ne.ne_gemm_trace(None, cap)
    try:
        for mode in (1, 2, 0):
            ne.ne_gemm_pair_halves(mode)
            o = empty_streams(M, R * Cc)
            for t in o:
                t.fill_(-1)
            ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, o, limb_bits=b)
            torch.cuda.synchronize()
            outs[mode] = o
    finally:
        ne.ne_gemm_pair_halves(0)
        ne.ne_gemm_trace(None, 0)
    for mode in (2, 0):
        assert all(torch.equal(x, y) for x, y in zip(outs[mode], outs[1])), mode
    out = outs[2]
    E = O.entangle(ocfg, A).reshape(M, R, K)
    rows = _band_rows(R, 128, seed=cap)
    ref = O.op_gemm(ocfg, E[:, rows], B.reshape(K, Cc))
    got = np.stack([out[m].view(R, Cc)[torch.from_numpy(rows).cuda()].cpu().numpy() for m in range(M)])
    assert (got == ref).all()
    x = np.random.default_rng(cap + 10).integers(-2, 2, size=Cc)   # |E (B x)| < 2^30 2^12 2^9 2^8 < 2^63
    bx = B.reshape(K, Cc) @ x
    for m in range(M):
        assert (out[m].cpu().numpy().reshape(R, Cc) @ x == E[m] @ bx).all(), m


def test_gemm_plain_i32(O):
    """The narrowest native baseline (plain one-digit GEMM, int32 products):
    every entry equal to A_m B (numpy on the same seeded inputs, exact: |A B|
    <= 1024 * 128 * 128 < 2^31), M = 3 streams of 256 x 512 at K = 1024."""
    M, R, Cc, K = 3, 256, 512, 1024
    A = gen(O, 84, 4, M, R * K, -128, 128)
    B = O.gen_uniform(84, 5, 0, -128, 128, K * Cc)
    planes = torch.empty(M * R * K, dtype=torch.int8, device="cuda")
    ne.ne_to_limbs(to_streams(A), 1, planes)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    out = [torch.full((R * Cc,), 7, dtype=torch.int32, device="cuda") for _ in range(M)]
    ne.ne_op_gemm_plain_i32(planes, Bt, R, Cc, K, out)
    ref = O.op_gemm(O.config_for(3, 64), A.reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    assert (to_np(out) == ref).all()


@pytest.mark.parametrize("cap", [0, 3])
def test_gemm_pair_one_digit(O, cap):
    """One int8 digit (plain data: the overhead baselines, ABFT's data GEMM)
    runs on the pair kernel's double-buffered mode (tile t in TMEM half
    t & 1): M = 4 streams of 1024 x 1024 at K = 2048 = 64 pair tiles, with
    the full grid and with the grid capped at 3 pairs (21-22 tiles each,
    both halves reused many times).  Sampled rows in every 32-lane group of
    128-row half (cycling) vs the oracle, whole output by Freivalds."""
    M, R, Cc, K = 4, 1024, 1024, 2048
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    assert ne.ne_gemm_kernel_for(cfg, 1, 8, R, Cc, K) == "pair"
    A = gen(O, 83, 4, M, R * K, -128, 128)
    B = O.gen_uniform(83, 5, 0, -128, 128, K * Cc)
    planes = torch.empty(M * R * K, dtype=torch.int8, device="cuda")
    ne.ne_to_limbs(to_streams(A), 1, planes)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    out = empty_streams(M, R * Cc)
    ne.ne_gemm_trace(None, cap)
    try:
        ne.ne_op_gemm_limbs(cfg, planes, 1, Bt, R, Cc, K, out, limb_bits=8)
        torch.cuda.synchronize()
    finally:
        ne.ne_gemm_trace(None, 0)
    A3 = A.reshape(M, R, K)
    rows = _band_rows_cyclic(R, 128)
    ref = O.op_gemm(ocfg, A3[:, rows], B.reshape(K, Cc))
    got = np.stack([out[m].view(R, Cc)[torch.from_numpy(rows).cuda()].cpu().numpy() for m in range(M)])
    assert (got == ref).all()
    x = np.random.default_rng(4).integers(-2 ** 16, 2 ** 16, size=Cc)   # |A (B x)| <= 2^11 2^7 2^34 < 2^63
    bx = B.reshape(K, Cc) @ x
    for m in range(M):
        assert (out[m].cpu().numpy().reshape(R, Cc) @ x == A3[m] @ bx).all(), m


def test_gemm_pair_short_k_many_tiles_sampled(O):
    """K = 2048 with >= 256 pair tiles also runs on the pair kernel (the
    paper's M = 8, N = 2000 shape class): rows sampled from every 256-row pair
    tile of every stream equal the oracle's products."""
    M, R, Cc, K = 8, 2048, 1024, 2048
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, 32)
    A = gen(O, 81, 4, M, R * K, -32, 32)
    B = O.gen_uniform(81, 5, 0, -32, 32, K * Cc)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    out = empty_streams(M, R * Cc)
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, limb_bits=b)
    assert ne.ne_gemm_kernel_for(cfg, L, b, R, Cc, K) == "pair"
    rows = _band_rows(R, 128)   # every 32-lane group (epilogue warp quarter) of every 128-row half
    E = O.entangle(ocfg, A).reshape(M, R, K)
    ref = O.op_gemm(ocfg, E[:, rows], B.reshape(K, Cc))
    got = np.stack([out[m].view(R, Cc)[torch.from_numpy(rows).cuda()].cpu().numpy() for m in range(M)])
    assert (got == ref).all()
    # the whole output: Freivalds with x in [-2^8, 2^8) (|E (B x)| <= 2^11 * 2^13 * 2^24 < 2^63)
    x = np.random.default_rng(1).integers(-2 ** 8, 2 ** 8, size=Cc)
    bx = B.reshape(K, Cc) @ x
    for m in range(M):
        assert (out[m].cpu().numpy().reshape(R, Cc) @ x == E[m] @ bx).all(), m


@pytest.mark.parametrize("max_clusters", [1, 3])
def test_gemm_capped_persistent_grid_and_trace(O, max_clusters):
    """The persistent scheduler with a capped grid (every CTA walks many work
    items, across both TMEM/stage phases) stays bit-exact; the debug trace
    (ne_gemm_trace) records, per CTA, accumulator-complete and epilogue-end
    times that are ordered within and across tiles."""
    M = 3
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, 127)
    R, Cc, K = 640, 1024, 384
    A = gen(O, 50, 4, M, R * K, -127, 128)
    B = O.gen_uniform(50, 5, 0, -128, 128, K * Cc)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    tr = torch.zeros(2 * max_clusters * 32 * 4, dtype=torch.int64, device="cuda")
    out = empty_streams(M, R * Cc)
    ne.ne_gemm_trace(tr, max_clusters)
    try:
        ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, limb_bits=b)
        torch.cuda.synchronize()
    finally:
        ne.ne_gemm_trace(None, 0)
    ref = O.op_gemm(ocfg, O.entangle(ocfg, A).reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    assert (to_np(out) == ref).all()
    t = tr.view(2 * max_clusters, 32, 4).cpu().numpy()
    n_items = M * (R // 128) * (Cc // 512)  # cluster work items (CTA pairs, 2 x 256 columns)
    for cta in range(2 * max_clusters):
        rows = [r for r in t[cta] if r[0] > 0]
        assert len(rows) == min(32, -(-(n_items - cta // 2) // max_clusters))
        for i, r in enumerate(rows):
            assert r[2] <= r[0] <= r[1]          # MMA start <= accumulators full <= epilogue end
            if i:
                assert rows[i - 1][0] <= r[2]   # single TMEM set: next tile starts after the previous is full


@pytest.mark.parametrize("M,a,b,R,Cc,K", [
    (3, 128, 127, 256, 512, 256),          # base-256 eps, 4 planes (one launch, the L = 4 kernel)
    (3, 1 << 10, 127, 256, 512, 384),      # split plan: c_m, c_{m-1} in 2 digits each at 0, 8, l, l + 8
    (3, 1 << 10, 128, 256, 512, 256),      # split plan x 2 B planes: reduce-add launches
    (3, 1 << 15, 1 << 15, 128, 256, 256),  # 5 eps planes (4 + 1 accumulators) x 3 B planes = 6 launches
    (4, 1 << 20, 1 << 15, 128, 256, 128),
    (8, 1 << 20, 1 << 10, 128, 384, 128),  # l = 8: eps digits overlap byte-aligned
])
def test_gemm_wide_range_plans(O, M, a, b, R, Cc, K):
    """The tensor-core GEMM over the certified operand range (missing in
    round 1): ne_gemm_plan_for's plan, the operand entangled into its digit
    planes, B into its digit planes, the multi-launch product — delta equal
    to the oracle's E B (mod 2^64 on both sides), the planes equal to the
    operands' digit expansions, and d_hat equal to the plain product when the
    product is certified (K a b <= hi)."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    plan = ne.ne_gemm_plan_for(cfg, a, b)
    A = gen(O, 90, 4, M, R * K, -a, a + 1)
    A[:, 0], A[:, 1] = a, -a
    B = O.gen_uniform(90, 5, 0, -b, b + 1, K * Cc)
    B[0], B[1] = b, -b
    planes = torch.empty(M * plan.LA * R * K, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_plan(cfg, to_streams(A), plan, planes, diag)
    Bt = torch.empty(plan.LB * Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b_planes(dev(B, torch.int32), K, Cc, plan.LB, Bt, diag)
    assert ne.diag_read(diag)["range_violations"] == 0
    E = O.entangle(ocfg, A)
    p = planes.cpu().numpy().astype(np.int64).reshape(M, plan.LA, R * K)
    assert (sum(p[:, i] << plan.a_shift[i] for i in range(plan.LA)) == E).all()
    q = Bt.cpu().numpy().astype(np.int64).reshape(plan.LB, Cc, K)
    assert (sum(q[j] << (8 * j) for j in range(plan.LB)).T.reshape(-1) == B).all()
    out = empty_streams(M, R * Cc)
    ne.ne_op_gemm_plan(cfg, planes, plan, Bt, R, Cc, K, out)
    ref = O.op_gemm(ocfg, E.reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    assert (to_np(out) == ref).all()
    if K * a * b <= O.dynamic_range(ocfg):
        d = empty_streams(M, R * Cc)
        ne.ne_disentangle_check(cfg, out, 0, d, None, diag)
        assert ne.diag_read(diag)["fault_positions"] == 0
        assert (to_np(d) == (A.reshape(M, R, K) @ B.reshape(K, Cc)).reshape(M, -1)).all()


def test_gemm_full_int64_operand_range(O):
    """ne_op_gemm (TC) over the widest operands: entangled A of full-range
    int32 inputs (8 base-256 digit planes) times full-range int32 B (5 digit
    planes): 16 tcgen05 launches accumulating into delta, equal to the
    oracle's wrapped int64 product (no operand range is refused)."""
    M, R, Cc, K = 3, 128, 256, 128
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    A = gen(O, 91, 4, M, R * K, -2 ** 31, 2 ** 31 - 1)
    B = O.gen_uniform(91, 5, 0, -2 ** 31, 2 ** 31 - 1, K * Cc)
    E = O.entangle(ocfg, A)
    ws = torch.empty(ne.ne_gemm_workspace(cfg, R, Cc, K, 8, 5), dtype=torch.int8, device="cuda")
    out = empty_streams(M, R * Cc)
    diag = ne.diag_new()
    ne.ne_op_gemm(cfg, to_streams(E, torch.int64), dev(B, torch.int32), R, Cc, K, out, L=8, ws=ws, diag=diag, LB=5)
    assert ne.diag_read(diag)["range_violations"] == 0
    ref = O.op_gemm(ocfg, E.reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    assert (to_np(out) == ref).all()


# ------------------------------------------------------------------ one-stream-per-GPU entry points (C5)
@pytest.mark.parametrize("M,L,bound", [(8, 2, 32), (3, 4, 64)])
def test_entangle_limbs_stream_and_gemm_stream(O, M, L, bound):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    R, Cc, K = 128, 256, 384
    A = gen(O, 4, 4, M, R * K, -bound, bound)
    B = O.gen_uniform(4, 5, 0, -bound, bound, K * Cc)
    E = O.entangle(ocfg, A)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    As = to_streams(A)
    for m in (0, M - 1):
        planes = torch.empty(L * R * K, dtype=torch.int8, device="cuda")
        ne.ne_entangle_limbs_stream(cfg, m, As[m], As[(m - 1) % M], L, planes)
        p = planes.cpu().numpy().astype(np.int64).reshape(L, -1)
        assert (sum(p[i] * 256 ** i for i in range(L)) == E[m]).all()
        out = torch.empty(R * Cc, dtype=torch.int64, device="cuda")
        ne.ne_op_gemm_limbs_stream(cfg, planes, L, Bt, R, Cc, K, out)
        ref = O.op_gemm(ocfg, E[m].reshape(R, K), B.reshape(K, Cc)).reshape(-1)
        assert (out.cpu().numpy() == ref).all()


@pytest.mark.parametrize("M,ndest,R,Cc,K", [(8, 8, 1024, 512, 256), (8, 4, 512, 1024, 384), (3, 2, 256, 768, 128),
                                           (3, 1, 384, 256, 256), (8, 8, 2048, 1024, 512)])
def test_gemm_scatter_fused_exchange(O, M, ndest, R, Cc, K):
    """ne_op_gemm_limbs_scatter: each stream's GEMM stores row block j straight
    into receiver j's buffer at that stream's slot (the position-major layout
    the check reads: [M][rows/ndest * cols] per receiver).  Receivers are
    local buffers here; the kernel only sees addresses (peer memory on a
    multi-GPU node).  Every receiver slice equals the oracle's product, and so
    does the optional full local copy."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, 32)
    A = gen(O, 60, 4, M, R * K, -32, 32)
    B = O.gen_uniform(60, 5, 0, -32, 32, K * Cc)
    E = O.entangle(ocfg, A)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    chunk = R // ndest * Cc
    recv = [torch.full((M * chunk,), -7, dtype=torch.int64, device="cuda") for _ in range(ndest)]
    As = to_streams(A)
    planes = torch.empty(L * R * K, dtype=torch.int8, device="cuda")
    local = empty_streams(M, R * Cc)
    for m in range(M):
        ne.ne_entangle_limbs_stream(cfg, m, As[m], As[(m - 1) % M], L, planes, limb_bits=b)
        ne.ne_op_gemm_limbs_scatter(cfg, planes, L, Bt, R, Cc, K, [recv[j][m * chunk:(m + 1) * chunk]
                                                                  for j in range(ndest)], limb_bits=b,
                                    local=local[m] if m % 2 else None)
    ref = O.op_gemm(ocfg, E.reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    for m in range(1, M, 2):   # the optional full local copy (what survivors exchange for recovery)
        assert (local[m].cpu().numpy() == ref[m]).all(), m
    for j in range(ndest):
        got = recv[j].view(M, chunk).cpu().numpy()
        assert (got == ref[:, j * chunk:(j + 1) * chunk]).all(), j
    # the receiver's slice disentangles and checks clean (what the C5 check runs on)
    d_out = empty_streams(M, chunk)
    diag = ne.diag_new()
    ne.ne_disentangle_check(cfg, [recv[ndest - 1][m * chunk:(m + 1) * chunk] for m in range(M)], 0, d_out, None, diag)
    plain = (A.reshape(M, R, K) @ B.reshape(K, Cc)).reshape(M, -1)[:, (ndest - 1) * chunk:]
    assert (to_np(d_out) == plain).all() and ne.diag_read(diag)["fault_positions"] == 0
    if R % (128 * 2 * ndest) != 0 and 2 * ndest <= 8:
        with pytest.raises(ne.NeError):   # row blocks that are not whole 128-row tiles: refused
            ne.ne_op_gemm_limbs_scatter(cfg, planes, L, Bt, R, Cc, K, [recv[0][:chunk // 2]] * (2 * ndest),
                                        limb_bits=b)


def test_c5_orchestration_single_gpu(O):
    """C5's host path on one GPU (world = 1: all 8 streams local), reduced size:
    entangle + tcgen05 GEMM per stream, check, kill stream 3, recover."""
    from paper_1604_04740_b200.dist import C5Plan, GpuBackend, c5_run

    plan = C5Plan(M=8, rows_total=8 * 128, cols=256, K=512, seed=4, bound=32, kill=3)
    res = c5_run(GpuBackend(plan.M, plan.bound), plan)
    assert res["flagged"] == 0 and res["checksum_ok"] is True
    B = O.gen_uniform(plan.seed, 5, 0, -32, 32, plan.K * plan.cols).reshape(plan.K, plan.cols)
    lo, d = res["check_slice"]
    lo2, d2 = res["recover_slice"]
    for m in range(plan.M):
        plain = (O.gen_uniform(plan.seed, 4, m, -32, 32, plan.rows * plan.K).reshape(plan.rows, plan.K) @ B).reshape(-1)
        assert (d[m].cpu().numpy() == plain).all() and (d2[m].cpu().numpy() == plain).all()


@pytest.mark.parametrize("symmetric", [False, True])
def test_c5_fused_exchange_single_gpu(O, symmetric):
    """C5 with exchange="fused" on one GPU: each stream's GEMM stores its
    output through ne_op_gemm_limbs_scatter into the receive window (a plain
    buffer, or torch symmetric memory rendezvoused over a one-rank NCCL group,
    the allocation the multi-GPU path stores into over NVLink), keeps the local
    copy for recovery; check, kill stream 3, recover — all bit-exact."""
    import socket

    import torch.distributed as dist

    from paper_1604_04740_b200.dist import C5Plan, GpuBackend, c5_run

    own_pg = False
    if symmetric and not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
        own_pg = True
    try:
        plan = C5Plan(M=8, rows_total=8 * 256, cols=512, K=256, seed=4, bound=32, kill=3)
        be = GpuBackend(plan.M, plan.bound)
        be.symmetric = symmetric
        res = c5_run(be, plan, exchange="fused")
        torch.cuda.synchronize()
    finally:
        if own_pg:
            dist.destroy_process_group()
    assert res["flagged"] == 0 and res["checksum_ok"] is True
    B = O.gen_uniform(plan.seed, 5, 0, -32, 32, plan.K * plan.cols).reshape(plan.K, plan.cols)
    lo, d = res["check_slice"]
    lo2, d2 = res["recover_slice"]
    for m in range(plan.M):
        plain = (O.gen_uniform(plan.seed, 4, m, -32, 32, plan.rows * plan.K).reshape(plan.rows, plan.K) @ B).reshape(-1)
        assert (d[m].cpu().numpy() == plain).all() and (d2[m].cpu().numpy() == plain).all()


# ------------------------------------------------------------------ BASELINE full sizes, bench launch config
def _band_rows(R, band=256, seed=0):
    """One row in every 32-row TMEM lane group of every `band`-row pair band:
    rows band*i + 32*q + j(i, q), so every epilogue warp quarter (q) of every
    pair tile row band is compared."""
    return np.array([band * i + 32 * q + (7 * i + 11 * q + seed) % 32
                     for i in range(R // band) for q in range(band // 32)])


def _band_rows_cyclic(R, band=256):
    """One row per `band`-row pair band, its 32-row lane group (CTA half and
    TMEM quarter) cycling with the band index: all 8 groups are covered
    every 8 bands."""
    return np.array([band * i + 32 * (i % (band // 32)) + (7 * i) % 32 for i in range(R // band)])


def _freivalds(O, got, A_rows, Bh, x):
    """got (R x C int64) == A (B x) for the test vector x (exact in int64:
    callers size x so that no product wraps)."""
    return (got @ x == A_rows @ (Bh @ x)).all()


@pytest.mark.parametrize("plan", ["pair", "base256"])
def test_c3_full_size_sampled(O, plan):
    """C3 at full size through the calls bench.py times.  plan "pair" is the
    bench default (ne_gemm_limb_plan: L = 2 digits in base 2^22), which the
    dispatch query confirms runs on the CTA-pair kernel (768 pair tiles over
    the SM pairs, many tiles per pair); "base256" is the L = 4 single-CTA
    path.  Checked against the oracle: one row in every 256-row band of
    every stream, its 32-row lane group cycling through all 8 (delta, d_hat);
    recovery of every r equal to d_hat in full; the whole d_hat by two Freivalds identities d_hat x == A_m (B x) (exact in
    int64), and the whole delta as the entanglement of d_hat (Eq. 15 on the
    oracle side), so every output position of every stream is covered."""
    M, n = 3, 4096
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    if plan == "pair":
        L, b = ne.ne_gemm_limb_plan(cfg, 64)
        assert (L, b) == (2, 22)
    else:
        L, b = ne.ne_gemm_limbs_for(cfg, 64), 8
        assert L == 4
    assert ne.ne_gemm_kernel_for(cfg, L, b, n, n, n) == ("pair" if plan == "pair" else "cta")
    A = [torch.empty(n * n, dtype=torch.int32, device="cuda") for _ in range(M)]
    for m in range(M):
        ne.ne_gen_uniform_i32(2, 4, m, -64, 64, A[m])
    B = torch.empty(n * n, dtype=torch.int32, device="cuda")
    ne.ne_gen_uniform_i32(2, 5, 0, -64, 64, B)
    planes = torch.empty(M * L * n * n, dtype=torch.int8, device="cuda")
    Bt = torch.empty(n * n, dtype=torch.int8, device="cuda")
    delta, dout = empty_streams(M, n * n), empty_streams(M, n * n)
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, A, L, planes, diag, b)
    ne.ne_gemm_prep_b(B, n, n, Bt, diag)
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, n, n, n, delta, b)
    bm = torch.empty(n * n // 32, dtype=torch.int32, device="cuda")
    ne.ne_disentangle_check(cfg, delta, 0, dout, bm, diag)
    d = ne.diag_read(diag)
    assert d["range_violations"] == 0 and d["fault_positions"] == 0 and int(bm.abs().sum()) == 0
    del planes, Bt
    Bh = O.gen_uniform(2, 5, 0, -64, 64, n * n).reshape(n, n)
    rows = _band_rows_cyclic(n)
    Ar = np.stack([np.stack([O.gen_uniform(2, 4, m, -64, 64, n, int(r) * n) for r in rows]) for m in range(M)])
    dref = O.op_gemm(ocfg, O.entangle(ocfg, Ar.reshape(M, -1)).reshape(M, len(rows), n), Bh)
    plain, _, nf = O.disentangle_check(ocfg, dref.reshape(M, -1), 0)
    assert nf == 0
    plain = plain.reshape(M, len(rows), n)
    ridx = torch.from_numpy(rows).cuda()
    assert (np.stack([t.view(n, n)[ridx].cpu().numpy() for t in delta]) == dref).all()
    assert (np.stack([t.view(n, n)[ridx].cpu().numpy() for t in dout]) == plain).all()
    for r in range(M):
        drec = empty_streams(M, n * n)
        ne.ne_recover(cfg, [None if m == r else delta[m] for m in range(M)], r, drec)
        assert all(torch.equal(x, y) for x, y in zip(drec, dout)), r
        del drec
    rng = np.random.default_rng(0)
    X = [rng.integers(-2 ** 20, 2 ** 20, size=n) for _ in range(2)]   # |A(Bx)| <= 2^12 * 2^6 * 2^38 < 2^63
    DH = to_np(dout)
    for m in range(M):
        Am = A[m].cpu().numpy().astype(np.int64).reshape(n, n)
        for x in X:
            assert _freivalds(O, DH[m].reshape(n, n), Am, Bh, x), m
    assert (to_np(delta) == O.entangle(ocfg, DH)).all()


def test_c4_full_size_sampled(O):
    """C4 at full size (M = 4, 2^28 positions): sampled output blocks vs the
    oracle recomputed from the generator at the permuted positions, for the
    fused gather kernel and for the op bench.py times (the partitioned
    scatter-reduce in its owned-run mode), whose delta, d_hat and bitmap
    equal the gather's in full."""
    M, n, Bk = 4, 1 << 28, 1024
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(M)]
    for m in range(M):
        ne.ne_gen_uniform_i32(3, 1, m, -(1 << 12), 1 << 12, c[m])
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ne.ne_gen_perm_i32(3, 6, perm)
    v = torch.empty(Bk, dtype=torch.int32, device="cuda")
    ne.ne_gen_uniform_i32(3, 7, 0, -(1 << 12), 1 << 12, v)
    eps = torch.empty(n * M, dtype=torch.int64, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_aos(cfg, c, eps, diag)
    del c
    nb = n // Bk
    delta, dout = empty_streams(M, nb), empty_streams(M, nb)
    bm = torch.empty(nb // 32, dtype=torch.int32, device="cuda")
    ne.ne_op_permute_inner_check(cfg, v, Bk, 0, dout, x_aos=eps, perm=perm, n=n, delta_out=delta, bitmap=bm,
                                 diag=diag)
    drec = empty_streams(M, nb)
    ne.ne_recover(cfg, [delta[0], delta[1], None, delta[3]], 2, drec)
    d = ne.diag_read(diag)
    assert d["range_violations"] == 0 and d["fault_positions"] == 0 and int(bm.abs().sum()) == 0
    assert all(torch.equal(a, b) for a, b in zip(dout, drec))
    # the timed form: partitioned scatter-reduce, owned runs (mode 1), the bench's r = 0
    assert ne.ne_permute_inner_plan(cfg, n, Bk)["mode"] == 1
    ws = torch.empty(ne.ne_permute_inner_workspace(cfg, n, Bk), dtype=torch.uint8, device="cuda")
    delta2, dout2 = empty_streams(M, nb), empty_streams(M, nb)
    bm2 = torch.full((nb // 32,), -1, dtype=torch.int32, device="cuda")
    diag2 = ne.diag_new()
    ne.ne_op_permute_inner_check_bucketed(cfg, eps, perm, v, Bk, 0, delta2, dout2, ws, bm2, diag2)
    del ws
    d2 = ne.diag_read(diag2)
    assert d2["range_violations"] == 0 and d2["fault_positions"] == 0 and int(bm2.abs().sum()) == 0
    assert all(torch.equal(a, b) for a, b in zip(delta, delta2)) and all(torch.equal(a, b) for a, b in zip(dout, dout2))
    vh = O.gen_uniform(3, 7, 0, -(1 << 12), 1 << 12, Bk)
    D, DH = to_np(delta), to_np(dout)
    for b in (0, 1, 12345, nb // 2 + 7, nb - 1):
        idx = O.gen_perm(3, 6, n, Bk, b * Bk)
        assert (perm[b * Bk:(b + 1) * Bk].cpu().numpy() == idx).all()
        cb = np.stack([np.array([O.gen_uniform(3, 1, m, -(1 << 12), 1 << 12, 1, int(p))[0] for p in idx])
                       for m in range(M)])
        e = O.entangle(ocfg, cb)
        dref = O.op_inner(ocfg, e, vh, Bk)[:, 0]
        assert (D[:, b] == dref).all()
        assert (DH[:, b] == O.op_inner(ocfg, cb, vh, Bk)[:, 0]).all()


def test_c5_full_size_single_gpu_protocol(O):
    """C5 at full size on one GPU (all 8 streams local), SURVEY §8(c) parity
    protocol 5: no position flagged; sampled entries of rows in every
    128-row tile band vs the oracle; two Freivalds identities d_hat_m x ==
    A_m (B x) over the WHOLE checked output of every stream (x in
    [-2^20, 2^20): |B x| <= 2^39, |A (B x)| <= 2^58, exact in int64); and the
    fail-stop of EVERY stream r = 0..7 recovered from the other 7 equals the
    checked d_hat in full (Props 1/3)."""
    import dataclasses

    from paper_1604_04740_b200.dist import C5Plan, GpuBackend, c5_setup, c5_step

    plan = C5Plan()
    M, K, cols, R = plan.M, plan.K, plan.cols, plan.rows
    be = GpuBackend(M, plan.bound)
    inp = c5_setup(be, plan)
    res = c5_step(be, plan, inp, verify=True)
    assert res["flagged"] == 0 and res["checksum_ok"] is True
    _, d = res["check_slice"]
    assert all(t.numel() == R * cols for t in d)
    chk = [t.clone() for t in d]
    for r in range(M):
        rr = c5_step(be, dataclasses.replace(plan, kill=r), inp, verify=False)
        _, drec = rr["recover_slice"]
        assert all(torch.equal(x, y) for x, y in zip(drec, chk)), r
    # whole-output Freivalds per stream
    Bh = O.gen_uniform(plan.seed, 5, 0, -32, 32, K * cols).reshape(K, cols)
    rng = np.random.default_rng(5)
    X = [rng.integers(-2 ** 20, 2 ** 20, size=cols) for _ in range(2)]
    BX = [Bh @ x for x in X]
    for m in range(M):
        Am = O.gen_uniform(plan.seed, 4, m, -32, 32, R * K).reshape(R, K)
        Dm = chk[m].cpu().numpy().reshape(R, cols)
        for x, bx in zip(X, BX):
            assert (Dm @ x == Am @ bx).all(), m
        del Am, Dm
    # sampled entries vs the oracle's own product
    cols_s = np.array([0, 1, 777, 8191, 16383])
    Bs = Bh[:, cols_s]
    rows = np.arange(0, R, 128) + (np.arange(R // 128) * 37) % 128
    for row in rows[::4]:
        Arow = np.stack([O.gen_uniform(plan.seed, 4, m, -32, 32, K, int(row) * K) for m in range(M)])
        plain = O.op_gemm(O.config_for(M, 64), Arow.reshape(M, 1, K), Bs).reshape(M, -1)
        got = np.stack([chk[m][int(row) * cols + cols_s].cpu().numpy() for m in range(M)])
        assert (got == plain).all(), row


# ------------------------------------------------------------------ ABFT comparison baseline (NEXT-1)
@pytest.mark.parametrize("M", [3, 4, 8])
@pytest.mark.parametrize("N", [16, 4096 + 16])
def test_abft_encode_check_recover(O, M, N):
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    rng = np.random.default_rng(M + N)
    c = rng.integers(-2 ** 20, 2 ** 20, size=(M, N))
    r = torch.empty(N, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_abft_encode(cfg, to_streams(c), r, diag)
    assert (r.cpu().numpy() == O.abft_encode(ocfg, c)).all()
    assert ne.diag_read(diag)["range_violations"] == 0
    big = np.full((M, N), 2 ** 30)  # the checksum's extra bits overflow int32 -> named range violation
    ne.ne_abft_encode(cfg, to_streams(big), r, diag)
    assert ne.diag_read(diag)["range_violations"] == N and ne.diag_read(diag)["first_bad"] == 0
    d = rng.integers(-2 ** 40, 2 ** 40, size=(M, N))
    e = d.sum(0)
    bad = d.copy()
    hit = rng.random(N) < 0.2
    for n in np.flatnonzero(hit):
        bad[rng.integers(0, M), n] ^= np.int64(1 << int(rng.integers(0, 63)))
    bm = torch.empty((N + 31) // 32, dtype=torch.int32, device="cuda")
    dg = ne.diag_new()
    ne.ne_abft_check(cfg, to_streams(bad, torch.int64), dev(e, torch.int64), bm, dg)
    flags, nf = O.abft_check(ocfg, bad, e)
    assert (bitmap_to_flags(bm, N) == flags).all() and ne.diag_read(dg)["fault_positions"] == nf == hit.sum()
    for lost in (0, M - 1):
        out = torch.empty(N, dtype=torch.int64, device="cuda")
        ds = to_streams(d, torch.int64)
        ne.ne_abft_recover(cfg, [None if m == lost else ds[m] for m in range(M)], dev(e, torch.int64), lost, out)
        assert (out.cpu().numpy() == d[lost]).all()


def test_abft_gemm_pipeline(O):
    """ABFT on tcgen05: plain data 1 int8 limb, checksum 2 limbs (|sum| <= 192),
    check clean, recovery of a lost stream by subtraction."""
    M, R, Cc, K = 3, 256, 256, 512
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    A = gen(O, 2, 4, M, R * K, -64, 64)
    B = O.gen_uniform(2, 5, 0, -64, 64, K * Cc)
    As = to_streams(A)
    Asum = torch.empty(R * K, dtype=torch.int32, device="cuda")
    diag = ne.diag_new()
    ne.ne_abft_encode(cfg, As, Asum, diag)
    pd = torch.empty(M * R * K, dtype=torch.int8, device="cuda")
    ps = torch.empty(2 * R * K, dtype=torch.int8, device="cuda")
    ne.ne_to_limbs(As, 1, pd, diag)
    ne.ne_to_limbs([Asum], 2, ps, diag)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt, diag)
    D = empty_streams(M, R * Cc)
    e = torch.empty(R * Cc, dtype=torch.int64, device="cuda")
    ne.ne_op_gemm_limbs(cfg, pd, 1, Bt, R, Cc, K, D)
    ne.ne_op_gemm_limbs_stream(cfg, ps, 2, Bt, R, Cc, K, e)
    ne.ne_abft_check(cfg, D, e, None, diag)
    dd = ne.diag_read(diag)
    assert dd["range_violations"] == 0 and dd["fault_positions"] == 0
    plain = (A.reshape(M, R, K) @ B.reshape(K, Cc)).reshape(M, -1)
    assert (to_np(D) == plain).all() and (e.cpu().numpy() == plain.sum(0)).all()
    out = torch.empty(R * Cc, dtype=torch.int64, device="cuda")
    ne.ne_abft_recover(cfg, [D[0], None, D[2]], e, 1, out)
    assert (out.cpu().numpy() == plain[1]).all()
    # the one-pass encode produces the same planes
    pd2, ps2 = torch.empty_like(pd), torch.empty_like(ps)
    ne.ne_abft_encode_limbs(cfg, As, pd2, 2, ps2, diag)
    assert torch.equal(pd, pd2) and torch.equal(ps, ps2) and ne.diag_read(diag)["range_violations"] == 0



# ------------------------------------------------------------------ base-2^l digit plan
@pytest.mark.parametrize("M,bound", [(3, 64), (3, 127), (4, 100), (5, 127)])
def test_base_l_digit_plan(O, M, bound):
    """The GEMM operand as two int8 digits in base 2^l (ne_gemm_limb_plan):
    entangle into digits, both GEMM entry points and the int64 split of
    ne_op_gemm agree with the oracle; a value outside the plan is flagged."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, bound)
    assert (L, b) == (2, cfg.l)
    R, Cc, K = 128, 256, 256
    A = gen(O, 6, 4, M, R * K, -bound, bound + 1)
    A[:, 0], A[:, 1] = bound, -bound
    B = O.gen_uniform(6, 5, 0, -128, 128, K * Cc)
    E = O.entangle(ocfg, A)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, diag, limb_bits=b)
    p = planes.cpu().numpy().astype(np.int64).reshape(M, L, -1)
    assert (p[:, 0] + p[:, 1] * 2 ** b == E).all() and ne.diag_read(diag)["range_violations"] == 0
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, Cc, Bt)
    ref = O.op_gemm(ocfg, E.reshape(M, R, K), B.reshape(K, Cc)).reshape(M, -1)
    out = empty_streams(M, R * Cc)
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, limb_bits=b)
    assert (to_np(out) == ref).all()
    out2 = empty_streams(M, R * Cc)
    ws = torch.empty(ne.ne_gemm_workspace(cfg, R, Cc, K, L), dtype=torch.int8, device="cuda")
    ne.ne_op_gemm(cfg, to_streams(E, torch.int64), dev(B, torch.int32), R, Cc, K, out2, L=L, ws=ws, diag=diag,
                  limb_bits=b)
    assert (to_np(out2) == ref).all()
    As = to_streams(A)
    pm = torch.empty(L * R * K, dtype=torch.int8, device="cuda")
    ne.ne_entangle_limbs_stream(cfg, 1, As[1], As[0], L, pm, diag, limb_bits=b)
    o1 = torch.empty(R * Cc, dtype=torch.int64, device="cuda")
    ne.ne_op_gemm_limbs_stream(cfg, pm, L, Bt, R, Cc, K, o1, limb_bits=b)
    assert (o1.cpu().numpy() == ref[1]).all()
    assert ne.diag_read(diag)["range_violations"] == 0
    big = A.copy()
    big[2 % M, 5] = 200   # |c| > 127: its two halves no longer fit int8
    ne.ne_entangle_limbs(cfg, to_streams(big), L, planes, diag, limb_bits=b)
    dd = ne.diag_read(diag)
    assert dd["range_violations"] >= 1


@pytest.mark.parametrize("M,align32", [(3, True), (3, False), (4, False), (5, True)])
def test_pair_digits_extremes_and_alignment(O, M, align32):
    """k_entangle_pair (the 32-bit two-digit path): digits equal the oracle's
    entangled value on representable entries; every non-representable entry
    (extreme int32 values included) is counted and the first one is named;
    16-B-only aligned streams take the 2 x 128-bit load path."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = 2, cfg.l
    N = 4096 + 16
    c = gen(O, 9, 1, M, N, -127, 128)
    specials = [2**31 - 1, -2**31, 200, -129, 128, -128, 127, 2**b, -(2**b), 2**b + 5, 2**(b - 1), -(2**(b - 1)) - 1]
    for k, v in enumerate(specials):
        c[k % M, 37 + 11 * k] = v
    E = O.entangle(ocfg, c)                        # exact (int64, w = 64)
    d0 = ((E + 2 ** (b - 1)) % 2 ** b) - 2 ** (b - 1)  # sext_b(E)
    d1 = (E - d0) >> b
    ok = (d0 >= -128) & (d0 <= 127) & (d1 >= -128) & (d1 <= 127)
    off = 0 if align32 else 4                      # int32 elements: 16-B offset
    streams = []
    for m in range(M):
        t = torch.zeros(N + 8, dtype=torch.int32, device="cuda")
        t[off:off + N] = torch.from_numpy(c[m].astype(np.int32)).cuda()
        streams.append(t[off:off + N])
    planes = torch.empty(M * L * N, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, streams, L, planes, diag, limb_bits=b)
    p = planes.cpu().numpy().astype(np.int64).reshape(M, L, N)
    assert (p[:, 0][ok] == d0[ok]).all() and (p[:, 1][ok] == d1[ok]).all()
    dd = ne.diag_read(diag)
    bad = np.flatnonzero((~ok).reshape(-1))
    assert dd["range_violations"] == len(bad) and len(bad) > 0
    assert dd["first_bad"] == bad.min()


@pytest.mark.parametrize("K,cols", [(64, 128), (192, 260), (16, 5), (4096, 384), (128, 64), (256, 192),
                                    (4096, 4160)])
def test_prep_b_ragged(O, K, cols):
    """B (K x cols int32) -> Bt (cols x K int8): full 128 x 64 tiles (K % 128 == 0,
    cols % 64 == 0; 4096 x 4160 = 2080 tiles, more than the persistent grid
    holds, so blocks walk several tiles through both shared buffers), partial
    64 x 128 tiles, scalar tail columns, and out-of-int8 entries counted with
    the first named."""
    B = O.gen_uniform(3, 5, 0, -128, 128, K * cols)
    B[7 % (K * cols)] = 300
    B[(K * cols) // 2] = -129
    Bt = torch.empty(cols * K, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, cols, Bt, diag)
    ref = B.reshape(K, cols).T.astype(np.int64)
    got = Bt.cpu().numpy().astype(np.int64).reshape(cols, K)
    okm = (ref >= -128) & (ref <= 127)
    assert (got[okm] == ref[okm]).all()
    dd = ne.diag_read(diag)
    bad = np.flatnonzero((B < -128) | (B > 127))
    assert dd["range_violations"] == len(bad) and dd["first_bad"] == bad.min()


# ------------------------------------------------------------------ GEMM with the fused check epilogue
@pytest.mark.parametrize("M,plan,bound,rows,cols,K,r", [
    (3, "pair", 64, 256, 512, 256, 0), (3, "pair", 127, 384, 256, 128, 2), (3, "b256", 64, 256, 384, 256, 1),
    (4, "pair", 100, 128, 256, 256, 3), (8, "b256", 32, 256, 256, 128, 5), (5, "pair", 100, 128, 128, 128, 4),
    (8, "pair", 32, 512, 1024, 256, 6), (3, "pair", 100, 1024, 2048, 256, 1)])
def test_gemm_limbs_check_fused(O, M, plan, bound, rows, cols, K, r):
    """ne_op_gemm_limbs_check == oracle GEMM (delta) + oracle disentangle/check
    (d_hat, flags, count, first) on clean data and with one stream's operand
    corrupted (a fault inside that stream's computation); the tile counters
    come back zeroed, and a second call on the same counters agrees.  M = 5
    exercises the unfused fallback."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    if plan == "pair":
        L, b = ne.ne_gemm_limb_plan(cfg, bound)
        assert (L, b) == (2, cfg.l)
    else:
        L, b = 4, 8
    A = np.stack([O.gen_uniform(8, 4, m, -bound, bound + 1, rows * K) for m in range(M)])
    B = O.gen_uniform(8, 5, 0, -128, 128, K * cols)
    planes = torch.empty(M * L * rows * K, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, to_streams(A), L, planes, diag, limb_bits=b)
    Bt = torch.empty(cols * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(B, torch.int32), K, cols, Bt, diag)
    cnt = torch.zeros(ne.ne_gemm_check_workspace(rows, cols) // 4, dtype=torch.int32, device="cuda")
    n = rows * cols
    for corrupt in (False, True, False):
        if corrupt:
            # a fault in stream s's operand: one digit of one row changes
            s, row, k = (r + 1) % M, rows // 2 + 3, 5
            planes.view(M, L, rows, K)[s, 0, row, k] += 1
        pl = planes.cpu().numpy().astype(np.int64).reshape(M, L, rows, K)
        E = sum(pl[:, i] * (2 ** (b * i)) for i in range(L))          # the operands the GPU consumes
        delta_ref = O.op_gemm(ocfg, E, B.reshape(K, cols)).reshape(M, -1)
        d_ref, f_ref, nf_ref = O.disentangle_check(ocfg, delta_ref, r)
        out, d_out = empty_streams(M, n), empty_streams(M, n)
        bm = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        dg = ne.diag_new()
        ne.ne_op_gemm_limbs_check(cfg, planes, L, Bt, rows, cols, K, out, r, d_out, cnt, bm, dg, limb_bits=b)
        torch.cuda.synchronize()
        assert (to_np(out) == delta_ref).all()
        assert (to_np(d_out) == d_ref).all()
        assert (bitmap_to_flags(bm, n) == f_ref).all()
        dd = ne.diag_read(dg)
        assert dd["fault_positions"] == nf_ref
        assert (nf_ref > 0) == corrupt
        if corrupt:
            assert dd["first_fault"] == int(np.flatnonzero(f_ref)[0])
            planes.view(M, L, rows, K)[s, 0, row, k] -= 1
        assert int(cnt.abs().sum()) == 0
    assert ne.diag_read(diag)["range_violations"] == 0


# ------------------------------------------------------------------ tensor-core (Toeplitz) convolution
@pytest.mark.parametrize("M,N,T,correlate,bound,block", [
    (3, 65536, 64, 0, 127, None), (3, 65536 + 77, 64, 1, 127, None), (4, 1000, 100, 0, 1000, None),
    (8, 5000, 4500, 0, 100, None), (3, 100, 300, 1, 127, None), (3, 384, 1, 0, 127, None),
    (5, 4096, 64, 1, 100, None), (3, 20000, 1000, 0, 127, None), (8, 70000, 700, 1, 100, 128),
    (3, 70000 + 5, 64, 0, 127, 256), (4, 600, 300, 1, 100, 256),
    # shift s0 mod N = 1, 2 (mod 4) for the vector-load entangle path
    (3, 4096, 2, 0, 127, None), (4, 8192, 67, 0, 100, None), (3, 100, 302, 0, 127, None),
    # Kpad >= 2048 at W = 256: the CTA-pair limb-major kernel (several pair row tiles, correlation, M = 4)
    (3, 70000 + 3, 2500, 1, 127, None), (4, 140000, 3000, 0, 100, None)])
def test_conv_tensor_core(O, M, N, T, correlate, bound, block):
    """ne_op_conv_limbs (tcgen05 Toeplitz GEMM + partial-block tail) equals the
    oracle's circular convolution / correlation of the entangled streams,
    bit for bit; the extended planes hold digit d of eps[(t - s0) mod N]."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    L, b = ne.ne_gemm_limb_plan(cfg, bound)
    c = gen(O, 11, 1, M, N, -bound, bound + 1)
    c[:, 0] = bound
    c[:, -1] = -bound
    g = O.gen_uniform(11, 3, 0, -128, 128, T)
    g[0] = -128
    eps = O.entangle(ocfg, c)
    bw, kp, plen = ne.ne_conv_geometry(N, T, L)
    if block is not None:
        bw = block
        kp = (T + bw - 1 + 127) // 128 * 128
        plen = (bw * ((N + bw - 1) // bw) + kp + bw - 1) // bw * bw
    assert bw == (256 if (T >= 256 and L <= 2) else 128) or block is not None
    assert kp % 128 == 0 and kp >= T + bw - 1 and plen % bw == 0
    planes = torch.empty(M * L * plen, dtype=torch.int8, device="cuda")
    Gt = torch.empty(bw * kp, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs_conv(cfg, to_streams(c), T, correlate, L, planes, diag, limb_bits=b, block=bw)
    ne.ne_conv_prep_taps(dev(g, torch.int32), correlate, Gt, diag, block=bw)
    out = empty_streams(M, N)
    ne.ne_op_conv_limbs(cfg, planes, L, Gt, N, T, correlate, out, limb_bits=b, block=bw)
    torch.cuda.synchronize()
    assert ne.diag_read(diag)["range_violations"] == 0
    assert (to_np(out) == O.op_conv(ocfg, eps, g, bool(correlate))).all()
    pl = planes.cpu().numpy().astype(np.int64).reshape(M, L, plen)
    rec = sum(pl[:, d] * (2 ** (b * d)) for d in range(L))
    s0 = 0 if correlate else T - 1
    idx = (np.arange(plen) - s0) % N
    assert (rec == eps[:, idx]).all()


def test_conv_tensor_core_range_violations(O):
    """Taps outside int8 and inputs outside the digit plan are counted once
    each and the first is named (tap index; m*N + n for inputs)."""
    M, N, T = 3, 3000, 70
    cfg = ne.ne_config_for(M)
    L, b = ne.ne_gemm_limb_plan(cfg, 127)
    c = gen(O, 12, 1, M, N, -100, 100)
    c[1, 17] = 300      # |c| > 127: not two int8 digits
    c[2, 5] = -129
    g = O.gen_uniform(12, 3, 0, -100, 100, T)
    g[9] = 128
    g[40] = -300
    bw, kp, plen = ne.ne_conv_geometry(N, T, L)
    planes = torch.empty(M * L * plen, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs_conv(cfg, to_streams(c), T, 0, L, planes, diag, limb_bits=b, block=bw)
    d = ne.diag_read(diag)
    # c[2,5] = -129 alone is still exact (d0 = -129 needs 9 bits: flagged), c[1,17] flagged;
    # the neighbour stream's digit d1 = c_{m-1} also leaves int8 for stream m+1
    E = O.entangle(O.config_for(M, 64), c)
    d0 = ((E + 2 ** (b - 1)) % 2 ** b) - 2 ** (b - 1)
    d1 = (E - d0) >> b
    bad = np.flatnonzero((~((d0 >= -128) & (d0 <= 127) & (d1 >= -128) & (d1 <= 127))).reshape(-1))
    assert d["range_violations"] == len(bad) and d["first_bad"] == bad.min()
    Gt = torch.empty(bw * kp, dtype=torch.int8, device="cuda")
    diag2 = ne.diag_new()
    ne.ne_conv_prep_taps(dev(g, torch.int32), 0, Gt, diag2, block=bw)
    d2 = ne.diag_read(diag2)
    assert d2["range_violations"] == 2 and d2["first_bad"] == 9


# ------------------------------------------------------------------ op + check fused in one kernel
@pytest.mark.parametrize("M,N,r", [(3, 4096, 0), (3, 4099, 2), (4, 1001, 3), (8, 777, 5), (5, 300, 1)])
def test_scale_add_check_fused(O, M, N, r):
    """ne_op_scale_add_check == oracle scale + add + disentangle/check (delta
    stored, d_hat, bitmap, count, first) on clean operands and with one
    stream's stored eps corrupted before the op (a fault in that stream)."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 13, 1, M, N, -2 ** 10, 2 ** 10)
    a = gen(O, 13, 2, M, N, -2 ** 10, 2 ** 10)
    E, A = O.entangle(ocfg, c), O.entangle(ocfg, a)
    for corrupt in (False, True):
        Ec = E.copy()
        if corrupt:
            Ec[(r + 1) % M, N // 3] ^= 1 << 40
            Ec[r, N - 1] ^= 12345
        D = O.op_add(ocfg, O.op_scale(ocfg, Ec, 37), A, 1)
        ref, flags, nf = O.disentangle_check(ocfg, D, r)
        x = to_streams(Ec, torch.int64)
        d_out = empty_streams(M, N)
        bm = torch.full(((N + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        dg = ne.diag_new()
        ne.ne_op_scale_add_check(cfg, x, 37, to_streams(A, torch.int64), r, d_out, bm, dg)
        assert (to_np(x) == D).all() and (to_np(d_out) == ref).all()
        assert (bitmap_to_flags(bm, N) == flags).all()
        d = ne.diag_read(dg)
        assert d["fault_positions"] == nf and (nf == 2) == corrupt
        if corrupt:
            assert d["first_fault"] == N // 3


@pytest.mark.parametrize("M,N,T,correlate,r,bit", [
    (3, 65536, 64, 0, 0, 7), (3, 1000, 64, 1, 1, 7), (4, 777, 1, 0, 2, 7), (8, 5000, 300, 1, 7, 7),
    (3, 50, 300, 0, 0, 7), (5, 2000, 64, 0, 4, 7), (3, 4096, 65, 0, 0, 40), (8, 3000, 257, 0, 3, 45),
    (3, 200000, 64, 0, 1, 7), (4, 160000, 33, 1, 0, 40)])
def test_conv_check_fused(O, M, N, T, correlate, r, bit):
    """ne_op_conv_check == oracle circular conv + disentangle/check, clean and
    with a corrupted stored eps word (flags exactly where the oracle's are);
    bit 40/45 puts a window value outside int32, so the 64-bit MAC path runs;
    odd T, T > 256 (several tap chunks), N up to 200 000."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 14, 1, M, N, -128, 128)
    g = O.gen_uniform(14, 3, 0, -128, 128, T)
    E = O.entangle(ocfg, c)
    for corrupt in (False, True):
        Ec = E.copy()
        if corrupt:
            Ec[(r + 2) % M, N // 2] ^= 1 << bit
        D = O.op_conv(ocfg, Ec, g, bool(correlate))
        ref, flags, nf = O.disentangle_check(ocfg, D, r)
        out, d_out = empty_streams(M, N), empty_streams(M, N)
        bm = torch.full(((N + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        dg = ne.diag_new()
        ne.ne_op_conv_check(cfg, to_streams(Ec, torch.int64), dev(g, torch.int32), out, r, d_out, bm, dg,
                            bool(correlate))
        assert (to_np(out) == D).all() and (to_np(d_out) == ref).all()
        assert (bitmap_to_flags(bm, N) == flags).all()
        d = ne.diag_read(dg)
        assert d["fault_positions"] == nf and (nf > 0) == corrupt


@pytest.mark.parametrize("M,sets,N", [(3, 2, 4096), (3, 2, 4099), (4, 3, 1001), (8, 4, 130), (5, 2, 77)])
def test_entangle_sets(O, M, sets, N):
    """Several independent stream sets in one launch: each set equals the
    oracle's entangle of that set; a range violation names (s*M + m)*N + n."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = np.concatenate([gen(O, 16 + s, 1, M, N, -1000, 1000) for s in range(sets)])
    eps = empty_streams(sets * M, N)
    diag = ne.diag_new()
    ne.ne_entangle_sets(cfg, to_streams(c), sets, eps, diag)
    got = to_np(eps)
    for s in range(sets):
        assert (got[s * M:(s + 1) * M] == O.entangle(ocfg, c[s * M:(s + 1) * M])).all()
    assert ne.diag_read(diag)["range_violations"] == 0
    hi = ne.ne_dynamic_range(cfg)
    c[(sets - 1) * M + 1, N - 1] = hi + 1 if hi < 2 ** 31 - 1 else c[0, 0]
    if hi < 2 ** 31 - 1:
        ne.ne_entangle_sets(cfg, to_streams(c), sets, eps, diag)
        d = ne.diag_read(diag)
        assert d["range_violations"] == 1 and d["first_bad"] == ((sets - 1) * M + 1) * N + N - 1


def test_gemm_int32_limb_sum_boundary():
    """The largest admissible K (130 944 < 2^31 / 2^14) with every digit and
    every B entry at -128: each int32 limb sum is K * 16384 = 2^31 - 2^21, the
    extreme the tensor-core accumulators must hold exactly; K = 131072 (sum
    2^31, which would wrap) is refused."""
    M, R, Cc, K = 3, 128, 128, 130944
    cfg = ne.ne_config_for(M)
    planes = torch.full((M * 1 * R * K,), -128, dtype=torch.int8, device="cuda")
    Bt = torch.full((Cc * K,), -128, dtype=torch.int8, device="cuda")
    out = empty_streams(M, R * Cc)
    ne.ne_op_gemm_limbs(cfg, planes, 1, Bt, R, Cc, K, out)
    torch.cuda.synchronize()
    assert all(bool((t == K * 16384).all()) for t in out)
    big = torch.empty(M * R * 131072, dtype=torch.int8, device="cuda")
    with pytest.raises(ne.NeError):
        ne.ne_op_gemm_limbs(cfg, big, 1, torch.empty(Cc * 131072, dtype=torch.int8, device="cuda"), R, Cc, 131072, out)


@pytest.mark.parametrize("M,Rt,Ct,Kt", [(3, 200, 300, 100), (8, 130, 1200, 200)])
def test_gemm_zero_padded_paper_shape(O, M, Rt, Ct, Kt):
    """The paper's GEMM shapes (2000 x N by N x 1200) are not tile
    multiples: operands zero-padded to (128, 256, 128) multiples give, in the
    true region, exactly the oracle's product of the unpadded operands, and the
    check on the padded output flags nothing."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    R, Cc, K = -(-Rt // 128) * 128, -(-Ct // 256) * 256, -(-Kt // 128) * 128
    L, b = ne.ne_gemm_limb_plan(cfg, 64)
    A = np.stack([O.gen_uniform(21, 4, m, -64, 64, Rt * Kt) for m in range(M)])
    B = O.gen_uniform(21, 5, 0, -64, 64, Kt * Ct)
    Ap = np.zeros((M, R, K), dtype=np.int64)
    Ap[:, :Rt, :Kt] = A.reshape(M, Rt, Kt)
    Bp = np.zeros((K, Cc), dtype=np.int64)
    Bp[:Kt, :Ct] = B.reshape(Kt, Ct)
    planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_entangle_limbs(cfg, to_streams(Ap.reshape(M, -1)), L, planes, diag, limb_bits=b)
    Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
    ne.ne_gemm_prep_b(dev(Bp.reshape(-1), torch.int32), K, Cc, Bt, diag)
    out, d_out = empty_streams(M, R * Cc), empty_streams(M, R * Cc)
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, limb_bits=b)
    ne.ne_disentangle_check(cfg, out, 0, d_out, None, diag)
    ref = O.op_gemm(ocfg, O.entangle(ocfg, A).reshape(M, Rt, Kt), B.reshape(Kt, Ct))
    got = to_np(out).reshape(M, R, Cc)
    assert (got[:, :Rt, :Ct] == ref).all() and (got[:, Rt:, :] == 0).all() and (got[:, :, Ct:] == 0).all()
    plain = A.reshape(M, Rt, Kt) @ B.reshape(Kt, Ct)
    assert (to_np(d_out).reshape(M, R, Cc)[:, :Rt, :Ct] == plain).all()
    d = ne.diag_read(diag)
    assert d["range_violations"] == 0 and d["fault_positions"] == 0


@pytest.mark.parametrize("M,N,T,correlate", [(3, 5000, 300, 0), (8, 4099, 64, 1), (3, 100, 257, 0)])
def test_abft_conv_tensor_core(O, M, N, T, correlate):
    """The paper's ABFT comparison on the tensor-core conv: data planes (one
    int8 digit), checksum planes (Eq. 4, base 256) in the extended layout, the
    plain Toeplitz conv of both, ABFT check (Eq. 6) and recovery ==
    the oracle's ABFT on the direct conv; a corrupted data output is flagged."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    c = gen(O, 22, 1, M, N, -128, 128)
    g = O.gen_uniform(22, 3, 0, -128, 128, T)
    bw, kp, plen = ne.ne_conv_geometry(N, T, 2)
    Ls = 2
    pdata = torch.empty(M * plen, dtype=torch.int8, device="cuda")
    psum = torch.empty(Ls * plen, dtype=torch.int8, device="cuda")
    Gt = torch.empty(bw * kp, dtype=torch.int8, device="cuda")
    diag = ne.diag_new()
    ne.ne_abft_encode_conv(cfg, to_streams(c), T, correlate, bw, pdata, Ls, psum, diag)
    ne.ne_conv_prep_taps(dev(g, torch.int32), correlate, Gt, diag, block=bw)
    d, e = empty_streams(M, N), empty_streams(1, N)
    ne.ne_op_conv_limbs_plain(M, pdata, 1, Gt, N, T, correlate, d, block=bw)
    ne.ne_op_conv_limbs_plain(1, psum, Ls, Gt, N, T, correlate, e, block=bw)
    torch.cuda.synchronize()
    assert ne.diag_read(diag)["range_violations"] == 0
    dref = O.op_conv(ocfg, c, g, bool(correlate))
    eref = O.op_conv(ocfg, O.abft_encode(ocfg, c)[None, :], g, bool(correlate))[0]
    assert (to_np(d) == dref).all() and (e[0].cpu().numpy() == eref).all()
    d[1][N // 2] += 5
    bm = torch.empty((N + 31) // 32, dtype=torch.int32, device="cuda")
    dg = ne.diag_new()
    ne.ne_abft_check(cfg, d, e[0], bm, dg)
    fref, nf = O.abft_check(ocfg, to_np(d), eref)
    assert (bitmap_to_flags(bm, N) == fref).all() and ne.diag_read(dg)["fault_positions"] == nf == 1
    rec = torch.empty(N, dtype=torch.int64, device="cuda")
    d[1][N // 2] -= 5
    ne.ne_abft_recover(cfg, [None if m == 2 else d[m] for m in range(M)], e[0], 2, rec)
    assert (rec.cpu().numpy() == dref[2]).all()


@pytest.mark.parametrize("M,r,W", [(4, 3, 32), (8, 5, 16), (5, 2, 24)])
def test_exhaustive_single_bit_injection_other_M(O, M, r, W):
    """a7 beyond C1: every single-bit flip of every stream in the first W
    outputs of a conv (M = 4, 8 and the generic-M kernel at M = 5, excluded
    stream r != 0) flags exactly its own position (Props 2/4, M l >= w), and
    d_hat at it equals the oracle's for the same corrupted word."""
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    N, T = 1024, 17
    c = gen(O, 23, 1, M, N, -100, 100)
    g = O.gen_uniform(23, 3, 0, -100, 100, T)
    delta = O.op_conv(ocfg, O.entangle(ocfg, c), g)
    trials = M * W * 64
    fw = torch.empty(trials, dtype=torch.int64, device="cuda")
    dh = torch.empty(trials * M, dtype=torch.int64, device="cuda")
    ne.ne_inject_sweep(cfg, to_streams(delta, torch.int64), W, r, fw, dh)
    fw = fw.cpu().numpy().view(np.uint64)
    dh = dh.cpu().numpy().reshape(trials, M)
    for t in range(trials):
        s, n, bit = t // (W * 64), (t // 64) % W, t % 64
        col = delta[:, n].copy()
        col[s] = np.int64(np.uint64(col[s]) ^ np.uint64(1 << bit))
        od, of = O.disentangle_one(ocfg, col, r)
        assert of == 1 and int(fw[t]) == (1 << n), (s, n, bit)
        assert (dh[t] == od).all(), (s, n, bit)


def test_diag_reset_and_accumulation(O):
    """ne_diag accumulates over calls (counts add, first_* keep the minimum)
    until ne_diag_reset restores {0, INT64_MAX, 0, INT64_MAX}."""
    M, N = 3, 4096
    cfg, ocfg = ne.ne_config_for(M), O.config_for(M, 64)
    d = torch.full((4,), 7, dtype=torch.int64, device="cuda")
    ne.ne_diag_reset(d)
    assert d.cpu().tolist() == [0, 2 ** 63 - 1, 0, 2 ** 63 - 1]
    c = gen(O, 70, 1, M, N, -100, 100)
    D = O.entangle(ocfg, c)
    out = empty_streams(M, N)
    for pos in (900, 300):
        Dc = D.copy()
        Dc[1, pos] ^= 1 << 9
        ne.ne_disentangle_check(cfg, to_streams(Dc, torch.int64), 0, out, None, d)
    r = ne.diag_read(d)
    assert r["fault_positions"] == 2 and r["first_fault"] == 300 and r["range_violations"] == 0
    ne.ne_diag_reset(d)
    assert ne.diag_read(d) == {"range_violations": 0, "first_bad": None, "fault_positions": 0, "first_fault": None}
