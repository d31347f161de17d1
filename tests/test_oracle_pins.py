"""Oracle pins (CPU): the oracle checked against what the paper and the
mathematics fix, never against itself.  SURVEY.md §8(c) checklist T1-T14.

Each test names the passage it pins.  A plausible mistake anywhere in the
oracle (dropped term, wrong sign or index, transposed operand) fails at least
one of these — see DESIGN.md §"Oracle pins" for the mistake -> test map.
"""
import math

import numpy as np
import pytest

from conftest import golden


def s64(v):
    """Python int -> the int64 with the same low 64 bits."""
    return ((v + 2 ** 63) % 2 ** 64) - 2 ** 63


# ---------------------------------------------------------------- T1 / T2
def test_T1_table2_w32(O):
    """Table II: (l, k, (M-2)l+k, w-ceil(log2 M)) for w = 32."""
    for (M, l, k, prop, abft), in golden("table2_w32.txt"):
        cfg = O.config_for(int(M), 32)
        assert (cfg.l, cfg.k) == (int(l), int(k))
        assert (int(M) - 2) * cfg.l + cfg.k == int(prop)
        assert 32 - math.ceil(math.log2(int(M))) == int(abft)


@pytest.mark.parametrize("M,l,k", [(3, 22, 20), (4, 16, 16), (5, 13, 12), (8, 8, 8), (11, 6, 4), (16, 4, 4), (32, 2, 2)])
def test_T2_config_w64(O, M, l, k):
    """Eq. 12 at w = 64; tie (21,21)/(22,20) at M = 3 -> larger l (F2)."""
    cfg = O.config_for(M, 64)
    assert (cfg.l, cfg.k) == (l, k)
    assert (M - 1) * cfg.l + cfg.k <= 64 and cfg.k <= cfg.l
    # invariants every configuration we use satisfies: M l >= w, (M-1)l+k = w
    assert M * cfg.l >= 64 and (M - 1) * cfg.l + cfg.k == 64


def test_T2_tie_is_real(O):
    """At w = 64, M = 3 both (21,21) and (22,20) reach (M-2)l+k = 42 (the tie F2 resolves)."""
    assert (3 - 2) * 21 + 21 == (3 - 2) * 22 + 20 == 42
    assert 2 * 21 + 21 <= 64 and 2 * 22 + 20 <= 64


def test_config_infeasible(O):
    """no (l,k) with l,k >= 1 when (M-1)+1 > w."""
    with pytest.raises(ValueError):
        O.config_for(40, 32)


# ---------------------------------------------------------------- T3
def test_T3_dynamic_range(O):
    """Eq. 11, Eq. 13, conservative min."""
    for (M, w, l, k, e11, e13, hi), in golden("dynamic_range.txt"):
        cfg = O.make_config(int(M), int(w), int(l), int(k))
        assert O.range_eq13(cfg) == int(e13)
        if e11 != "-":
            assert O.range_eq11(cfg) == int(e11)
        assert O.dynamic_range(cfg) == int(hi)


def test_T3_range_is_sufficient_bound(O):
    """Eq. 13 keeps entangled values inside w bits: (2^l+1) hi <= 2^(w-1)-1 and
    hi < 2^((M-1)l-1) (the two limits the disentangling needs), every config."""
    for M in (3, 4, 5, 8, 11, 16):
        for w in (32, 64):
            cfg = O.config_for(M, w)
            hi = O.dynamic_range(cfg)
            assert (2 ** cfg.l + 1) * hi <= 2 ** (w - 1) - 1
            assert hi < 2 ** ((M - 1) * cfg.l - 1)


def test_T3_degenerate_l1(O):
    """F4: Eq. 13 is 0 at (M=32, w=32, l=1): the configuration admits only 0."""
    assert O.dynamic_range(O.config_for(32, 32)) == 0


# ---------------------------------------------------------------- T4 / T5
def test_T4_entangle_hand_values(O):
    """Eq. 7 / Eq. 15 hand values."""
    for (M, w, l, k), c, eps in golden("entangle_hand.txt"):
        cfg = O.make_config(int(M), int(w), int(l), int(k))
        out = O.entangle(cfg, np.array([int(v) for v in c]).reshape(-1, 1))
        assert out.ravel().tolist() == [int(v) for v in eps]


def test_T4_entangle_is_circulant_operator(O):
    """Eq. 14: column n of eps is E c with E = I + S_l P (P the cyclic shift);
    check against an explicit integer matrix product (numpy) for M = 5."""
    cfg = O.config_for(5, 64)
    rng = np.random.default_rng(1)
    c = rng.integers(-1000, 1000, size=(5, 7))
    E = np.eye(5, dtype=np.int64)
    for m in range(5):
        E[m, (m - 1) % 5] = 2 ** cfg.l
    assert (O.entangle(cfg, c) == E @ c).all()


def test_T5_eq10_trace(O):
    """Eq. 10 hand trace: (6145, 2050, 4099), r = 0 -> (1, 2, 3), no flag."""
    (d0, d1, d2, r), (dtemp,), dh = golden("eq10_trace.txt")[0]
    cfg = O.make_config(3, 32, 11, 10)
    out, flag = O.disentangle_one(cfg, [int(d0), int(d1), int(d2)], int(r))
    assert out.tolist() == [int(v) for v in dh]
    assert flag == 0
    # the trace's d_temp is delta2 - S_l{delta1}; the sign reading R1 hinges on it
    assert int(d2) - int(d1) * 2 ** 11 == int(dtemp)


# ---------------------------------------------------------------- T6 / T12
@pytest.mark.parametrize("w", [32, 64])
def test_T6_roundtrip_every_r(O, w):
    """Props 1/3 + S:120: disentangle(entangle(c), r) = c for every r, M."""
    rng = np.random.default_rng(w)
    for M in (3, 4, 5, 8, 11, 16, 32):
        cfg = O.config_for(M, w)
        hi = O.dynamic_range(cfg)
        if hi == 0:
            continue
        c = rng.integers(-hi, hi + 1, size=(M, 1000))
        c[:, 0], c[:, 1], c[:, 2] = hi, -hi, 0  # extremes
        c[:, 3] = [hi if m % 2 else -hi for m in range(M)]
        eps = O.entangle(cfg, c)
        for r in range(M):
            d, flags, nf = O.disentangle_check(cfg, eps, r)
            assert (d == c).all(), (M, w, r)
            assert nf == 0


def test_T12_recovery_each_stream(O):
    """Props 1/3: drop any one stream, recover all."""
    rng = np.random.default_rng(12)
    for M in range(3, 9):
        cfg = O.config_for(M, 64)
        hi = O.dynamic_range(cfg)
        c = rng.integers(-hi, hi + 1, size=(M, 100))
        eps = O.entangle(cfg, c)
        for r in range(M):
            rows = [None if m == r else eps[m] for m in range(M)]
            assert (O.recover(cfg, rows, r) == c).all()
        with pytest.raises(ValueError):
            O.recover(cfg, [None, None] + [eps[m] for m in range(2, M)], 0)


# ---------------------------------------------------------------- T8
def _np_conv(x, g, correlate=False):
    N = x.shape[-1]
    out = np.zeros_like(x)
    for j, gj in enumerate(g):
        out += gj * np.roll(x, -j if correlate else j, axis=-1)
    return out


def test_T8_op_definitions_vs_numpy(O):
    """Each oracle op at w = 64 equals the textbook/library routine (numpy)."""
    cfg = O.config_for(3, 64)
    rng = np.random.default_rng(8)
    x = rng.integers(-1000, 1000, size=(3, 50))
    g = rng.integers(-50, 50, size=50)
    assert (O.op_scale(cfg, x, 37) == 37 * x).all()
    assert (O.op_scale(cfg, x, g=g) == x * g).all()
    a = rng.integers(-1000, 1000, size=(3, 50))
    assert (O.op_add(cfg, x, a, 1) == x + a).all()
    assert (O.op_add(cfg, x, a, -1) == x - a).all()
    v = rng.integers(-9, 9, size=10)
    inner = O.op_inner(cfg, x, v, 10)
    assert (inner == (x.reshape(3, 5, 10) * v).sum(-1)).all()
    # ragged last block: N = 50, block 16 -> blocks of 16,16,16,2 (v indexed i mod 16)
    v16 = rng.integers(-9, 9, size=16)
    ref = np.stack([[np.dot(x[m, b:b + 16], v16[: len(x[m, b:b + 16])]) for b in range(0, 50, 16)] for m in range(3)])
    assert (O.op_inner(cfg, x, v16, 16) == ref).all()
    h = rng.integers(-9, 9, size=7)
    assert (O.op_outer(cfg, x, h) == x[:, :, None] * h[None, None, :]).all()
    taps = rng.integers(-20, 20, size=8)
    assert (O.op_conv(cfg, x, taps) == _np_conv(x, taps)).all()
    assert (O.op_conv(cfg, x, taps, correlate=True) == _np_conv(x, taps, True)).all()
    A = rng.integers(-64, 64, size=(3, 6, 9))
    B = rng.integers(-64, 64, size=(9, 5))
    assert (O.op_gemm(cfg, A, B) == A @ B).all()
    perm = rng.permutation(50)
    assert (O.op_permute(x, perm) == x[:, perm]).all()


def test_T8_spec_conv_examples(O):
    """S:236-237 style trivial conv cases: delta kernel, all-ones kernel."""
    cfg = O.config_for(3, 64)
    x = np.array([[1, 2, 3]] * 3)
    assert (O.op_conv(cfg, x, [1, 0, 0]) == x).all()
    assert (O.op_conv(cfg, x, [1, 1, 1]) == 6).all()


@pytest.mark.parametrize("M", [3, 4, 8])
@pytest.mark.parametrize("w", [32, 64])
def test_T8_homomorphism(O, M, w):
    """P:380-386 / Eq. 9: disentangle(op(entangle(c))) = op(c), op from the
    plain definition in Z (numpy), for every op kind."""
    cfg = O.config_for(M, w)
    hi = O.dynamic_range(cfg)
    rng = np.random.default_rng(M * 100 + w)
    cfg64 = O.config_for(M, 64)
    for trial in range(20):
        N = int(rng.integers(1, 40))
        B = max(1, hi // 64)
        c = rng.integers(-B, B + 1, size=(M, N))
        eps = O.entangle(cfg, c)

        def check(delta, plain):
            for r in (0, M - 1, int(rng.integers(0, M))):
                d, _, nf = O.disentangle_check(cfg, delta, r)
                assert nf == 0 and (d == plain).all(), (M, w, r)

        # scale by a constant and elementwise by g
        s = int(rng.integers(-8, 9))
        check(O.op_scale(cfg, eps, s), s * c)
        g = rng.integers(-8, 9, size=N)
        check(O.op_scale(cfg, eps, g=g), c * g)
        # add: per-stream addend entangled by E (R10); shared g self-entangled
        a = rng.integers(-B, B + 1, size=(M, N))
        check(O.op_add(cfg, eps, O.entangle(cfg, a), 1), c + a)
        check(O.op_add(cfg, eps, O.entangle(cfg, a), -1), c - a)
        gs = rng.integers(-B, B + 1, size=N)
        gent = O.entangle_shared(cfg, gs)
        check(O.op_add(cfg, eps, np.broadcast_to(gent, (M, N)).copy(), 1), c + gs)
        # permutation commutes with entanglement
        perm = rng.permutation(N)
        assert (O.op_permute(eps, perm) == O.entangle(cfg, c[:, perm])).all()
        check(O.op_permute(eps, perm), c[:, perm])
        # inner / outer / conv / gemm with small operands keep outputs in range
        v = rng.integers(-4, 5, size=4)
        c4 = rng.integers(-(hi // 32 + 1), hi // 32 + 1, size=(M, N))
        e4 = O.entangle(cfg, c4)
        ip = O.op_inner(cfg, e4, v, 4)
        d, _, nf = O.disentangle_check(cfg, ip, 0)
        assert nf == 0 and (d == O.op_inner(cfg64, c4, v, 4)).all()
        h = rng.integers(-4, 5, size=3)
        ou = O.op_outer(cfg, e4, h).reshape(M, -1)
        d, _, nf = O.disentangle_check(cfg, ou, 1)
        assert nf == 0 and (d.reshape(M, N, 3) == c4[:, :, None] * h).all()
        taps = rng.integers(-2, 3, size=min(N, 5))
        for corr in (False, True):
            cv = O.op_conv(cfg, e4, taps, corr)
            d, _, nf = O.disentangle_check(cfg, cv, 0)
            assert nf == 0 and (d == _np_conv(c4, taps, corr)).all()
        K = 4
        A = rng.integers(-(hi // 64 + 1), hi // 64 + 1, size=(M, 3, K))
        Bm = rng.integers(-4, 5, size=(K, 2))
        EA = O.entangle(cfg, A.reshape(M, -1)).reshape(M, 3, K)
        Cm = O.op_gemm(cfg, EA, Bm).reshape(M, -1)
        d, _, nf = O.disentangle_check(cfg, Cm, 2 % M)
        assert nf == 0 and (d.reshape(M, 3, 2) == A @ Bm).all()


def test_T8_self_entangle_spec_example(O):
    """S:184 / P:507-511: add_const 5 at l = 11 -> operand 5*2048+5 = 10245."""
    cfg = O.make_config(3, 32, 11, 10)
    assert O.entangle_shared(cfg, [5]).tolist() == [10245]


# ---------------------------------------------------------------- T9 / T11 / T13
@pytest.mark.parametrize("M", [3, 8])
@pytest.mark.parametrize("w", [32, 64])
def test_T9_single_bit_detection_after_conv(O, M, w):
    """Props 2/4 (proofs P:1190-1258): every single-bit
    flip of one delta_s[n] after an LSB op is flagged, at n only."""
    cfg = O.config_for(M, w)
    hi = O.dynamic_range(cfg)
    rng = np.random.default_rng(9)
    N = 16
    taps = rng.integers(-3, 4, size=4)
    c = rng.integers(-(hi // 16), hi // 16 + 1, size=(M, N))
    delta = O.op_conv(cfg, O.entangle(cfg, c), taps)
    d0, _, nf = O.disentangle_check(cfg, delta, 0)
    assert nf == 0
    for s in range(M):
        for n in range(N):
            for bit in range(w):
                bad = delta.copy()
                bad[s, n] = O.wrap(cfg, s64(int(bad[s, n]) ^ (1 << bit)))
                d, flags, nf = O.disentangle_check(cfg, bad, 0)
                assert nf == 1 and flags[n] == 1, (s, n, bit)


def test_T11_no_false_positives(O):
    """Zero flags on 10^4 clean in-range blocks."""
    rng = np.random.default_rng(11)
    for M in (3, 4, 8):
        cfg = O.config_for(M, 64)
        hi = O.dynamic_range(cfg)
        c = rng.integers(-hi, hi + 1, size=(M, 10000))
        for r in range(M):
            _, _, nf = O.disentangle_check(cfg, O.entangle(cfg, c), r)
            assert nf == 0


def test_T13_detection_limit_double_fault(O):
    """two co-located faults can pass: delta1 += x, delta2 += x 2^l."""
    cfg = O.config_for(3, 64)
    eps = O.entangle(cfg, np.array([[5], [7], [9]]))[:, 0]
    bad = eps.copy()
    bad[1] += 3
    bad[2] += 3 * 2 ** cfg.l
    d, flag = O.disentangle_one(cfg, bad, 0)
    assert flag == 0 and d.tolist() == [5, 10, 9]


def test_F2_tiebreak_counterexample(O):
    """F2: with l = 21 the single-word corruption delta2 -= 2^63+1 is silent
    (the aliasing period 2^(Ml)+1 = 2^63+1 is reachable); with l = 22 it is flagged."""
    c = np.array([[5], [7], [9]])
    for l, k, silent in ((21, 21, True), (22, 20, False)):
        cfg = O.make_config(3, 64, l, k)
        eps = O.entangle(cfg, c)[:, 0]
        bad = eps.copy()
        bad[2] = s64(int(bad[2]) - (2 ** 63 + 1))
        d, flag = O.disentangle_one(cfg, bad, 0)
        if silent:
            assert flag == 0 and d.tolist() != [5, 7, 9]
        else:
            assert flag == 1


def test_check_uses_2w_bits(O):
    """F3: a mod-2^64 compare would miss faults at M=3, l=22 (R can reach 2^65);
    the oracle's exact compare flags every single-bit flip of streams 1, 2 in
    bits 20-21 / 42-43 where the truncated compare is blind."""
    cfg = O.config_for(3, 64)
    rng = np.random.default_rng(3)
    hi = O.dynamic_range(cfg)
    for _ in range(50):
        c = rng.integers(-hi, hi + 1, size=(3, 1))
        eps = O.entangle(cfg, c)[:, 0]
        for s, bits in ((1, (20, 21)), (2, (42, 43))):
            for bit in bits:
                bad = eps.copy()
                bad[s] ^= 1 << bit
                _, flag = O.disentangle_one(cfg, bad, 0)
                assert flag == 1


# ---------------------------------------------------------------- T14
def test_T14_range_assertion(O):
    """range error naming (m, n): first_bad = m*N + n; +-hi accepted."""
    cfg = O.config_for(3, 64)
    hi = O.dynamic_range(cfg)
    c = np.zeros((3, 10), dtype=np.int64)
    c[0, 0], c[2, 9] = hi, -hi
    assert O.range_check(c, hi) == (0, -1)
    c[1, 4] = hi + 1
    c[2, 2] = -hi - 1
    assert O.range_check(c, hi) == (2, 1 * 10 + 4)


def test_T14_certify_examples(O):
    """S:190-195 certification arithmetic; config bounds of BASELINE C1-C5 are admissible."""
    cfg = O.config_for(3, 32)
    hi = O.dynamic_range(cfg)
    assert O.certify("conv", 10000, 100) == 1_000_000 <= hi
    assert O.certify("conv", 20000, 100) == 2_000_000 > hi
    assert O.certify("permute", 12345, 0) == 12345
    h3, h4, h8 = (O.dynamic_range(O.config_for(M, 64)) for M in (3, 4, 8))
    c1 = O.certify("add", O.certify("scale", 2 ** 10, 37), 2 ** 10)   # 37 c + a
    assert c1 == 38912 <= h3
    assert O.certify("conv", 128, 64 * 128) == 2 ** 20 <= h3          # C2
    assert 2 ** 20 > O.dynamic_range(O.config_for(3, 32))             # C2 needs w = 64
    assert O.certify("gemm", 64, 4096 * 64) == 2 ** 24 <= h3           # C3
    assert O.certify("inner", 2 ** 12, 1024 * 2 ** 12) == 2 ** 34 <= h4  # C4
    assert O.certify("gemm", 32, 16384 * 32) == 2 ** 24 <= h8          # C5


# ---------------------------------------------------------------- generator
def test_generator_splitmix_reference_value(O):
    """gen/ne_gen.h: mix(0) is SplitMix64's published first output for state 0
    (0xE220A8397B1DCDAF); uniform values stay in [lo, hi)."""
    import ctypes

    lib = O.lib()
    # u(seed=0,tag=0,stream=0,idx) = mix(mix(0) + idx); probe mix(0) through the
    # uniform map with span 2^32: value = lo + (u >> 32)
    first = 0xE220A8397B1DCDAF
    key = first  # ne_gen_key(0,0,0) = mix(0)
    # reproduce u for idx = 0 by the definition with Python integers
    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
        return z ^ (z >> 31)
    assert mix(0) == first
    vals = O.gen_uniform(0, 0, 0, 0, 2 ** 32, 4)
    assert vals.tolist() == [mix(key + i) >> 32 for i in range(4)]
    x = O.gen_uniform(7, 1, 2, -1024, 1024, 100000)
    assert x.min() >= -1024 and x.max() < 1024 and abs(x.mean()) < 20
    del lib, ctypes


@pytest.mark.parametrize("n", [1, 2, 3, 17, 1000, 4096, 65537])
def test_generator_perm_is_bijection(O, n):
    p = O.gen_perm(3, 6, n)
    assert np.array_equal(np.sort(p), np.arange(n))
    if n >= 1000:
        assert (p != np.arange(n)).mean() > 0.99
