"""CPU oracle for arXiv 1604.04740 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package.  The
product path (``paper_1604_04740_b200``) never does, and fails loudly when its
CUDA library is missing instead of falling back here.

This module is argument marshalling (numpy <-> ctypes) around ``liboracle.so``
(plain C11 + __int128, ``oracle/ne_oracle.c``); all arithmetic is in the C.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# NE_ORACLE_UBSAN=1: the same sources built with -fsanitize=undefined and
# -fno-sanitize-recover=all (any undefined behaviour aborts the process); the
# CPU suite runs the oracle pins against it (tests/test_oracle_ubsan.py)
UBSAN = os.environ.get("NE_ORACLE_UBSAN") == "1"
_SO = os.path.join(_HERE, "liboracle_ubsan.so" if UBSAN else "liboracle.so")


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in ("ne_oracle.c", "or_selftest.c", "ne_oracle.h")]
    srcs.append(os.path.join(_HERE, "..", "gen", "ne_gen.h"))
    if force or not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in srcs):
        cc = os.environ.get("CC", "gcc")
        flags = ["-O2", "-std=gnu11", "-Wall", "-fPIC", "-pthread"]
        if UBSAN:   # the system gcc carries libubsan
            cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else cc
            flags = ["-O1", "-g", "-std=gnu11", "-Wall", "-fPIC", "-pthread", "-fsanitize=undefined",
                     "-fno-sanitize-recover=all"]
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call([cc, *flags, "-shared", "-o", tmp, os.path.join(_HERE, "ne_oracle.c"),
                               os.path.join(_HERE, "or_selftest.c")])
        os.replace(tmp, _SO)
    return _SO


class Config(C.Structure):
    _fields_ = [("M", C.c_int32), ("w", C.c_int32), ("l", C.c_int32), ("k", C.c_int32)]

    def __repr__(self) -> str:  # pragma: no cover - debugging aid
        return f"Config(M={self.M}, w={self.w}, l={self.l}, k={self.k})"


_lib = None
_P64 = C.POINTER(C.c_int64)
_PU8 = C.POINTER(C.c_uint8)
_PCFG = C.POINTER(Config)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        sig = {
            "or_config_for": (C.c_int32, [C.c_int32, C.c_int32, _PCFG]),
            "or_dynamic_range": (C.c_int64, [_PCFG]),
            "or_range_eq11": (C.c_int64, [_PCFG]),
            "or_range_eq13": (C.c_int64, [_PCFG]),
            "or_wrap": (C.c_int64, [_PCFG, C.c_int64]),
            "or_range_check": (C.c_int64, [_P64, C.c_int64, C.c_int64, _P64]),
            "or_entangle": (None, [_PCFG, _P64, C.c_int64, _P64]),
            "or_entangle_shared": (None, [_PCFG, _P64, C.c_int64, _P64]),
            "or_op_scale": (None, [_PCFG, _P64, C.c_int64, C.c_int64, C.c_int64, _P64]),
            "or_op_add": (None, [_PCFG, _P64, _P64, C.c_int64, C.c_int64, C.c_int32]),
            "or_op_inner": (None, [_PCFG, _P64, C.c_int64, C.c_int64, _P64, C.c_int64, C.c_int64, _P64]),
            "or_op_outer": (None, [_PCFG, _P64, C.c_int64, C.c_int64, _P64, C.c_int64, _P64]),
            "or_op_conv": (None, [_PCFG, _P64, C.c_int64, C.c_int64, _P64, C.c_int64, C.c_int32, _P64]),
            "or_op_gemm": (None, [_PCFG, _P64, C.c_int64, C.c_int64, _P64, C.c_int64, _P64]),
            "or_set_threads": (None, [C.c_int32]),
            "or_max_threads": (C.c_int32, []),
            "or_op_permute": (None, [_P64, C.c_int64, C.c_int64, _P64, _P64]),
            "or_disentangle_one": (C.c_int32, [_PCFG, _P64, C.c_int32, _P64, C.c_int32]),
            "or_disentangle_check": (C.c_int64, [_PCFG, _P64, C.c_int64, C.c_int32, _P64, _PU8]),
            "or_recover": (C.c_int32, [_PCFG, C.POINTER(_P64), C.c_int64, C.c_int32, _P64]),
            "or_certify": (C.c_int64, [C.c_int32, C.c_int64, C.c_int64]),
            "or_abft_encode": (None, [_PCFG, _P64, C.c_int64, _P64]),
            "or_abft_check": (C.c_int64, [_PCFG, _P64, _P64, C.c_int64, _PU8]),
            "or_abft_recover": (C.c_int32, [_PCFG, C.POINTER(_P64), _P64, C.c_int64, C.c_int32, _P64]),
            "or_gen_uniform": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_int64, _P64]),
            "or_gen_perm": (None, [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64, C.c_int64, _P64]),
            "or_selftest_roundtrip_box": (C.c_int64, [_PCFG, C.c_int64, _P64]),
            "or_selftest_word_sweep": (C.c_int64, [_PCFG, _P64, _P64, _P64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_P64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


# ------------------------------------------------------------------ a0
def config_for(M: int, w: int) -> Config:
    cfg = Config()
    if lib().or_config_for(M, w, C.byref(cfg)) != 0:
        raise ValueError(f"configuration error: no feasible (l,k) for M={M}, w={w}")
    return cfg


def make_config(M: int, w: int, l: int, k: int) -> Config:
    return Config(M, w, l, k)


def dynamic_range(cfg: Config) -> int:
    return int(lib().or_dynamic_range(C.byref(cfg)))


def range_eq11(cfg: Config) -> int:
    return int(lib().or_range_eq11(C.byref(cfg)))


def range_eq13(cfg: Config) -> int:
    return int(lib().or_range_eq13(C.byref(cfg)))


def wrap(cfg: Config, x: int) -> int:
    return int(lib().or_wrap(C.byref(cfg), int(x)))


def range_check(x, hi: int):
    x = _i64(x).ravel()
    fb = C.c_int64()
    n = lib().or_range_check(_p(x), x.size, hi, C.byref(fb))
    return int(n), int(fb.value)


def certify(op: str, in_bound: int, operand: int) -> int:
    code = {"scale": 0, "add": 1, "inner": 2, "conv": 2, "gemm": 2, "permute": 3}[op]
    return int(lib().or_certify(code, in_bound, operand))


# ------------------------------------------------------------------ a1/a2
def entangle(cfg: Config, c) -> np.ndarray:
    c = _i64(c)
    assert c.ndim == 2 and c.shape[0] == cfg.M
    out = np.empty_like(c)
    lib().or_entangle(C.byref(cfg), _p(c), c.shape[1], _p(out))
    return out


def entangle_shared(cfg: Config, g) -> np.ndarray:
    g = _i64(g).ravel()
    out = np.empty_like(g)
    lib().or_entangle_shared(C.byref(cfg), _p(g), g.size, _p(out))
    return out


# ------------------------------------------------------------------ a3
def op_scale(cfg: Config, x, s: int = 1, g=None) -> np.ndarray:
    x = _i64(x).copy()
    rows, N = x.reshape(-1, x.shape[-1]).shape
    gp = None
    if g is not None:
        g = _i64(g)
        gp = _p(g)
    lib().or_op_scale(C.byref(cfg), _p(x), rows, N, int(s), gp)
    return x


def op_add(cfg: Config, x, a, sign: int = 1) -> np.ndarray:
    x = _i64(x).copy()
    a = _i64(a)
    assert a.shape == x.shape
    rows, N = x.reshape(-1, x.shape[-1]).shape
    lib().or_op_add(C.byref(cfg), _p(x), _p(a), rows, N, int(sign))
    return x


def op_inner(cfg: Config, x, v, block: int) -> np.ndarray:
    x = _i64(x)
    v = _i64(v).ravel()
    rows, N = x.shape
    nb = (N + block - 1) // block
    out = np.empty((rows, nb), dtype=np.int64)
    lib().or_op_inner(C.byref(cfg), _p(x), rows, N, _p(v), v.size, block, _p(out))
    return out


def op_outer(cfg: Config, x, h) -> np.ndarray:
    x = _i64(x)
    h = _i64(h).ravel()
    rows, N1 = x.shape
    out = np.empty((rows, N1, h.size), dtype=np.int64)
    lib().or_op_outer(C.byref(cfg), _p(x), rows, N1, _p(h), h.size, _p(out))
    return out


def op_conv(cfg: Config, x, g, correlate: bool = False) -> np.ndarray:
    x = _i64(x)
    g = _i64(g).ravel()
    rows, N = x.shape
    out = np.empty_like(x)
    lib().or_op_conv(C.byref(cfg), _p(x), rows, N, _p(g), g.size, int(correlate), _p(out))
    return out


def op_gemm(cfg: Config, A, B) -> np.ndarray:
    """A: (..., rows, K) stack of stream sub-blocks; B: (K, cols)."""
    A = _i64(A)
    B = _i64(B)
    K, cols = B.shape
    lead = A.shape[:-1]
    A2 = A.reshape(-1, K)
    out = np.empty((A2.shape[0], cols), dtype=np.int64)
    lib().or_op_gemm(C.byref(cfg), _p(A2), A2.shape[0], K, _p(B), cols, _p(out))
    return out.reshape(*lead, cols)


def set_threads(n: int) -> None:
    """OpenMP threads of op_gemm (1 = the single-core baseline)."""
    lib().or_set_threads(int(n))


def max_threads() -> int:
    return int(lib().or_max_threads())


def op_permute(x, perm) -> np.ndarray:
    x = _i64(x)
    perm = _i64(perm).ravel()
    rows, N = x.shape
    assert perm.size == N
    out = np.empty_like(x)
    lib().or_op_permute(_p(x), rows, N, _p(perm), _p(out))
    return out


# ------------------------------------------------------------------ a4-a6
def disentangle_one(cfg: Config, delta, r: int = 0, check: bool = True):
    d = _i64(delta).ravel()
    out = np.empty(cfg.M, dtype=np.int64)
    f = lib().or_disentangle_one(C.byref(cfg), _p(d), int(r), _p(out), int(check))
    return out, int(f)


def disentangle_check(cfg: Config, delta, r: int = 0):
    delta = _i64(delta)
    M, N = delta.shape
    assert M == cfg.M
    out = np.empty_like(delta)
    flags = np.zeros(N, dtype=np.uint8)
    nf = lib().or_disentangle_check(C.byref(cfg), _p(delta), N, int(r), _p(out),
                                    flags.ctypes.data_as(_PU8))
    return out, flags, int(nf)


def recover(cfg: Config, delta_rows, r: int) -> np.ndarray:
    """delta_rows: list of M arrays (or None for the absent stream)."""
    M = cfg.M
    keep = [None if d is None else _i64(d) for d in delta_rows]
    N = next(d.size for d in keep if d is not None)
    ptrs = (_P64 * M)(*[(_P64() if d is None else _p(d)) for d in keep])
    out = np.empty((M, N), dtype=np.int64)
    rc = lib().or_recover(C.byref(cfg), ptrs, N, int(r), _p(out))
    if rc != 0:
        raise ValueError("unrecoverable: more than one stream absent, or the absent stream is not r")
    return out


# ------------------------------------------------------------------ ABFT baseline (Eqs. 3-6)
def abft_encode(cfg: Config, c) -> np.ndarray:
    c = _i64(c)
    out = np.empty(c.shape[1], dtype=np.int64)
    lib().or_abft_encode(C.byref(cfg), _p(c), c.shape[1], _p(out))
    return out


def abft_check(cfg: Config, d, e):
    d, e = _i64(d), _i64(e).ravel()
    flags = np.zeros(e.size, dtype=np.uint8)
    nf = lib().or_abft_check(C.byref(cfg), _p(d), _p(e), e.size, flags.ctypes.data_as(_PU8))
    return flags, int(nf)


def abft_recover(cfg: Config, d_rows, e, r: int) -> np.ndarray:
    keep = [None if x is None else _i64(x) for x in d_rows]
    e = _i64(e).ravel()
    ptrs = (_P64 * cfg.M)(*[(_P64() if x is None else _p(x)) for x in keep])
    out = np.empty(e.size, dtype=np.int64)
    if lib().or_abft_recover(C.byref(cfg), ptrs, _p(e), e.size, int(r), _p(out)) != 0:
        raise ValueError("unrecoverable: exactly stream r must be absent")
    return out


# ------------------------------------------------------------------ inputs
def gen_uniform(seed: int, tag: int, stream: int, lo: int, hi: int, count: int, offset: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    lib().or_gen_uniform(seed, tag, stream, lo, hi, offset, count, _p(out))
    return out


def gen_perm(seed: int, tag: int, n: int, count: int | None = None, offset: int = 0) -> np.ndarray:
    count = n if count is None else count
    out = np.empty(count, dtype=np.int64)
    lib().or_gen_perm(seed, tag, n, offset, count, _p(out))
    return out


# ------------------------------------------------------------------ self-test loops
def selftest_roundtrip_box(cfg: Config, H: int):
    n = C.c_int64()
    fails = lib().or_selftest_roundtrip_box(C.byref(cfg), H, C.byref(n))
    return int(fails), int(n.value)


def selftest_word_sweep(cfg: Config, c):
    c = _i64(c).ravel()
    miss, sil = C.c_int64(), C.c_int64()
    tried = lib().or_selftest_word_sweep(C.byref(cfg), _p(c), C.byref(miss), C.byref(sil))
    return int(tried), int(miss.value), int(sil.value)
