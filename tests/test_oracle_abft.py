"""Pins of the oracle's ABFT baseline (Eqs. 3-6): SPEC worked
values, linearity of the checksum under every LSB op, single-fault detection,
the compensating double-fault limit, and recovery by subtraction."""
import numpy as np

from conftest import golden


def test_abft_spec_values(O):
    for (kind,), vals, (exp,) in golden("abft_spec.txt"):
        v = [int(x) for x in vals]
        if kind == "encode":
            cfg = O.config_for(len(v), 64)
            assert O.abft_encode(cfg, np.array(v).reshape(-1, 1)).tolist() == [int(exp)]
        elif kind == "recover0":  # M=3, stream 0 lost; vals = d1, d2, e
            cfg = O.config_for(3, 64)
            out = O.abft_recover(cfg, [None, [v[0]], [v[1]]], [v[2]], 0)
            assert out.tolist() == [int(exp)]
        else:  # M=4, stream 1 lost; vals = d0, d2, d3, e
            cfg = O.config_for(4, 64)
            out = O.abft_recover(cfg, [[v[0]], None, [v[1]], [v[2]]], [v[3]], 1)
            assert out.tolist() == [int(exp)]
    cfg = O.config_for(3, 64)
    r = O.abft_encode(cfg, np.array([[1], [2], [3]]))
    assert O.op_scale(cfg, r.reshape(1, 1), 2).ravel().tolist() == [12]


def test_abft_linearity_detection_recovery(O):
    rng = np.random.default_rng(7)
    for M in (3, 4, 8):
        cfg = O.config_for(M, 64)
        c = rng.integers(-1000, 1000, size=(M, 64))
        r = O.abft_encode(cfg, c)
        assert (r == c.sum(0)).all()
        taps = rng.integers(-5, 6, size=7)
        full = np.vstack([c, r])
        cfgp = O.config_for(M + 1, 64)  # the op runs on M+1 streams (Eq. 5)
        d = O.op_conv(cfgp, full, taps)
        flags, nf = O.abft_check(cfg, d[:M], d[M])
        assert nf == 0
        for s in range(M + 1):           # any single stream of the M+1, any bit
            for bit in (0, 17, 62):
                bad = d.copy()
                bad[s, 9] ^= np.int64(1 << bit)
                flags, nf = O.abft_check(cfg, bad[:M], bad[M])
                assert nf == 1 and flags[9] == 1
        bad = d.copy()                   # compensating double fault evades (SPEC detection limit)
        bad[0, 3] += 5
        bad[1, 3] -= 5
        assert O.abft_check(cfg, bad[:M], bad[M])[1] == 0
        for lost in range(M):
            rows = [None if m == lost else d[m] for m in range(M)]
            assert (O.abft_recover(cfg, rows, d[M], lost) == d[lost]).all()
