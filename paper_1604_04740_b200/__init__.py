"""paper_1604_04740_b200 — B200-native numerical entanglement (arXiv 1604.04740).

Thin Python binding of ``libne.so`` (C ABI declared in ``include/ne.h``): the
functions below carry the C names and only marshal arguments (torch CUDA
tensors -> device pointers, the current CUDA stream).  Every step of the hot
path runs in the library's sm_100a kernels.  There is no CPU fallback: if the
library or a CUDA device is missing, the calls raise.

Layout conventions: a stream set is a list of M 1-D torch tensors (int32 for
plain inputs, int64 for entangled data / outputs), each contiguous and 16-byte
aligned; ``diag`` is a device int64 tensor of 4 words (``ne_diag``).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import torch

from ._build import LIB, build  # noqa: F401  (build() is what __graft_entry__.build calls)

NE_MAX_M = 32
STATUS = {0: "NE_OK", 1: "NE_EINVAL", 2: "NE_ECONFIG", 3: "NE_ERANGE", 4: "NE_EINDEX",
          5: "NE_EUNRECOVERABLE", 6: "NE_ECUDA", 7: "NE_ENOTSUP"}
NE_GEMM_TC_I8, NE_GEMM_IMAD64, NE_GEMM_IMAD32W = 0, 1, 2
NE_OP_SCALE, NE_OP_ADD, NE_OP_LINEAR, NE_OP_PERMUTE = 0, 1, 2, 3

# every symbol include/ne.h and include/ne_gendev.h declare (checked by tests)
EXPORTS = (
    "ne_config_for", "ne_dynamic_range", "ne_certify", "ne_gemm_limbs_for", "ne_gemm_limb_plan", "ne_diag_reset",
    "ne_entangle", "ne_entangle_sets", "ne_entangle_sets_w32", "ne_entangle_aos", "ne_entangle_limbs", "ne_entangle_stream", "ne_entangle_shared",
    "ne_entangle_limbs_stream", "ne_op_gemm_limbs_stream",
    "ne_op_scale", "ne_op_add", "ne_op_scale_add", "ne_op_inner", "ne_op_outer", "ne_op_conv", "ne_op_permute",
    "ne_gemm_workspace", "ne_op_gemm", "ne_gemm_prep_b", "ne_op_gemm_limbs",
    "ne_gemm_plan_for", "ne_entangle_plan", "ne_gemm_prep_b_planes", "ne_op_gemm_plan", "ne_op_gemm_plain_i32",
    "ne_gemm_check_workspace", "ne_op_gemm_limbs_check", "ne_gemm_trace", "ne_gemm_pair_schedule", "ne_gemm_pair_halves", "ne_gemm_kernel_for", "ne_op_gemm_limbs_scatter",
    "ne_conv_geometry", "ne_entangle_limbs_conv", "ne_conv_prep_taps", "ne_op_conv_limbs",
    "ne_op_scale_add_check", "ne_op_conv_check", "ne_op_scale_add_check_w32",
    "ne_entangle_w32", "ne_op_scale_add_w32", "ne_disentangle_check_w32", "ne_recover_w32", "ne_inject_sweep_w32",
    "ne_entangle_aos_w32", "ne_op_permute_inner_check_w32",
    "ne_disentangle_check", "ne_recover", "ne_op_permute_inner_check", "ne_op_permute_inner_stream", "ne_permute_inner_workspace", "ne_permute_inner_plan", "ne_op_permute_inner_check_bucketed",
    "ne_inject", "ne_inject_sweep", "ne_gen_uniform_i32", "ne_gen_perm_i32",
    "ne_abft_encode", "ne_abft_encode_limbs", "ne_abft_encode_conv", "ne_op_conv_limbs_plain", "ne_to_limbs", "ne_abft_check", "ne_abft_recover",
)


class NeError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} returned {STATUS.get(status, status)}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("M", C.c_int32), ("w", C.c_int32), ("l", C.c_int32), ("k", C.c_int32)]

    def __repr__(self) -> str:
        return f"ne_config(M={self.M}, w={self.w}, l={self.l}, k={self.k})"


class GemmPlan(C.Structure):  # ne_gemm_plan
    _fields_ = [("kind", C.c_int32), ("LA", C.c_int32), ("digit_bits", C.c_int32), ("LB", C.c_int32),
                ("a_shift", C.c_int32 * 8)]

    def __repr__(self) -> str:
        return (f"ne_gemm_plan(kind={'split' if self.kind else 'eps'}, LA={self.LA}, digit_bits={self.digit_bits}, "
                f"LB={self.LB}, a_shift={list(self.a_shift)[:self.LA]})")


class Streams(C.Structure):  # ne_streams / ne_cstreams / ne_cstreams32 (same ABI)
    _fields_ = [("s", C.c_void_p * NE_MAX_M)]


_lib = None
_PCFG = C.POINTER(Config)
_VP = C.c_void_p
_I64, _I32, _U64, _SZ = C.c_int64, C.c_int32, C.c_uint64, C.c_size_t

_SIGS = {
    "ne_config_for": [_I32, _I32, _PCFG],
    "ne_dynamic_range": [_PCFG, C.POINTER(_I64)],
    "ne_certify": [_PCFG, C.c_int, _I64, _I64, C.POINTER(_I64)],
    "ne_gemm_limbs_for": [_PCFG, _I64],
    "ne_gemm_limb_plan": [_PCFG, _I64, C.POINTER(_I32)],
    "ne_diag_reset": [_VP, _VP],
    "ne_entangle": [_PCFG, Streams, _I64, Streams, _VP, _VP],
    "ne_entangle_sets": [_PCFG, Streams, _I32, _I64, Streams, _VP, _VP],
    "ne_entangle_sets_w32": [_PCFG, Streams, _I32, _I64, Streams, _VP, _VP],
    "ne_entangle_aos": [_PCFG, Streams, _I64, _VP, _VP, _VP],
    "ne_entangle_limbs": [_PCFG, Streams, _I64, _I32, _I32, _VP, _VP, _VP],
    "ne_entangle_stream": [_PCFG, _I32, _VP, _VP, _VP, _I64, _VP, _VP],
    "ne_entangle_shared": [_PCFG, _VP, _VP, _I64, _VP],
    "ne_entangle_limbs_stream": [_PCFG, _I32, _VP, _VP, _I64, _I32, _I32, _VP, _VP, _VP],
    "ne_op_gemm_limbs_stream": [_PCFG, _VP, _I32, _I32, _VP, _I64, _I64, _I64, _VP, _VP],
    "ne_op_scale": [_PCFG, Streams, _I64, _I64, _VP, _VP],
    "ne_op_add": [_PCFG, Streams, Streams, _I64, _I32, _VP],
    "ne_op_scale_add": [_PCFG, Streams, _I64, _I64, _VP, Streams, _I32, _VP],
    "ne_op_inner": [_PCFG, Streams, _I64, _VP, _I64, _I64, Streams, _VP],
    "ne_op_outer": [_PCFG, Streams, _I64, _VP, _I64, Streams, _VP],
    "ne_op_conv": [_PCFG, Streams, _I64, _VP, _I32, _I32, Streams, _VP],
    "ne_op_permute": [_PCFG, Streams, _VP, _I64, Streams, _VP],
    "ne_gemm_workspace": [_PCFG, _I64, _I64, _I64, _I32, _I32, C.POINTER(_SZ)],
    "ne_op_gemm": [_PCFG, Streams, _VP, _I64, _I64, _I64, C.c_int, _I32, _I32, _I32, Streams, _VP, _SZ, _VP, _VP],
    "ne_gemm_plan_for": [_PCFG, _I64, _I64, C.POINTER(GemmPlan)],
    "ne_entangle_plan": [_PCFG, Streams, _I64, C.POINTER(GemmPlan), _VP, _VP, _VP],
    "ne_gemm_prep_b_planes": [_VP, _I64, _I64, _I32, _VP, _VP, _VP],
    "ne_op_gemm_plan": [_PCFG, _VP, C.POINTER(GemmPlan), _VP, _I64, _I64, _I64, Streams, _VP],
    "ne_op_gemm_plain_i32": [_I32, _VP, _VP, _I64, _I64, _I64, Streams, _VP],
    "ne_gemm_prep_b": [_VP, _I64, _I64, _VP, _VP, _VP],
    "ne_op_gemm_limbs": [_PCFG, _VP, _I32, _I32, _VP, _I64, _I64, _I64, Streams, _VP],
    "ne_op_scale_add_check": [_PCFG, Streams, _I64, _I64, _VP, Streams, _I32, _I32, Streams, _VP, _VP, _VP],
    "ne_op_conv_check": [_PCFG, Streams, _I64, _VP, _I32, _I32, Streams, _I32, Streams, _VP, _VP, _VP],
    "ne_op_scale_add_check_w32": [_PCFG, Streams, _I64, _I32, _VP, Streams, _I32, _I32, Streams, _VP, _VP, _VP],
    "ne_entangle_w32": [_PCFG, Streams, _I64, Streams, _VP, _VP],
    "ne_op_scale_add_w32": [_PCFG, Streams, _I64, _I32, _VP, C.POINTER(Streams), _I32, _VP],
    "ne_disentangle_check_w32": [_PCFG, Streams, _I64, _I32, Streams, _VP, _VP, _VP],
    "ne_recover_w32": [_PCFG, Streams, _I64, _I32, Streams, _VP],
    "ne_inject_sweep_w32": [_PCFG, Streams, _I64, _I32, _VP, _VP, _VP],
    "ne_entangle_aos_w32": [_PCFG, Streams, _I64, _VP, _VP, _VP],
    "ne_op_permute_inner_check_w32": [_PCFG, _VP, _VP, _I64, _VP, _I64, _I64, _I32, Streams, Streams, _VP, _VP, _VP],
    "ne_conv_geometry": [_I64, _I32, _I32, C.POINTER(_I32), C.POINTER(_I64), C.POINTER(_I64)],
    "ne_entangle_limbs_conv": [_PCFG, Streams, _I64, _I32, _I32, _I32, _I32, _I32, _VP, _VP, _VP],
    "ne_conv_prep_taps": [_VP, _I32, _I32, _I32, _VP, _VP, _VP],
    "ne_op_conv_limbs": [_PCFG, _VP, _I32, _I32, _I32, _VP, _I64, _I32, _I32, Streams, _VP],
    "ne_gemm_check_workspace": [_I64, _I64, C.POINTER(_SZ)],
    "ne_gemm_trace": [_VP, _I32],
    "ne_gemm_pair_schedule": [_I64, _I64, C.POINTER(_I64)],
    "ne_gemm_pair_halves": [_I32],
    "ne_gemm_kernel_for": [_PCFG, _I32, _I32, _I64, _I64, _I64, C.POINTER(_I32)],
    "ne_op_gemm_limbs_scatter": [_PCFG, _VP, _I32, _I32, _VP, _I64, _I64, _I64, Streams, _I32, _VP, _VP],
    "ne_op_gemm_limbs_check": [_PCFG, _VP, _I32, _I32, _VP, _I64, _I64, _I64, Streams, _I32, Streams, _VP, _VP, _VP,
                               _VP],
    "ne_disentangle_check": [_PCFG, Streams, _I64, _I32, Streams, _VP, _VP, _VP],
    "ne_recover": [_PCFG, Streams, _I64, _I32, Streams, _VP],
    "ne_permute_inner_workspace": [_PCFG, _I64, _I64, C.POINTER(_SZ)],
    "ne_permute_inner_plan": [_PCFG, _I64, _I64, C.POINTER(_I32), C.POINTER(_I32), C.POINTER(_I32),
                              C.POINTER(_I32), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64)],
    "ne_op_permute_inner_check_bucketed": [_PCFG, _VP, _VP, _I64, _VP, _I64, _I64, _I32, Streams, Streams, _VP, _VP,
                                           _VP, _SZ, _VP],
    "ne_op_permute_inner_check": [_PCFG, Streams, _VP, _I32, _VP, _I64, _VP, _I64, _I64, _I32,
                                  Streams, Streams, _VP, _VP, _VP],
    "ne_op_permute_inner_stream": [_PCFG, _VP, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _VP, _VP],
    "ne_inject": [_VP, _I64, _U64, _VP],
    "ne_abft_encode_conv": [_PCFG, Streams, _I64, _I32, _I32, _I32, _VP, _I32, _VP, _VP, _VP],
    "ne_op_conv_limbs_plain": [_I32, _VP, _I32, _I32, _I32, _VP, _I64, _I32, _I32, Streams, _VP],
    "ne_abft_encode": [_PCFG, Streams, _I64, _VP, _VP, _VP],
    "ne_to_limbs": [Streams, _I32, _I64, _I32, _VP, _VP, _VP],
    "ne_abft_encode_limbs": [_PCFG, Streams, _I64, _VP, _I32, _VP, _VP, _VP],
    "ne_abft_check": [_PCFG, Streams, _VP, _I64, _VP, _VP, _VP],
    "ne_abft_recover": [_PCFG, Streams, _VP, _I64, _I32, _VP, _VP],
    "ne_inject_sweep": [_PCFG, Streams, _I64, _I32, _VP, _VP, _VP],
    "ne_gen_uniform_i32": [_U64, C.c_uint32, C.c_uint32, _I64, _I64, _I64, _I64, _VP, _VP],
    "ne_gen_perm_i32": [_U64, C.c_uint32, _I64, _VP, _VP],
}


def lib() -> C.CDLL:
    """Load libne.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _lib = L
    return _lib


def _call(name: str, *args) -> int:
    st = getattr(lib(), name)(*args)
    if st != 0:
        raise NeError(name, st)
    return st


def _stream():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1604_04740_b200 needs a CUDA device (no CPU fallback)")
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None, dtype=None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensors only")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("contiguous tensors only")
    return C.c_void_p(t.data_ptr())


def _streams(ts: Sequence[torch.Tensor | None], dtype) -> Streams:
    s = Streams()
    for i, t in enumerate(ts):
        s.s[i] = None if t is None else _ptr(t, dtype).value
    return s


# ------------------------------------------------------------------ a0 (host)
def ne_config_for(M: int, w: int = 64) -> Config:
    cfg = Config()
    _call("ne_config_for", M, w, C.byref(cfg))
    return cfg


def ne_dynamic_range(cfg: Config) -> int:
    hi = C.c_int64()
    _call("ne_dynamic_range", C.byref(cfg), C.byref(hi))
    return hi.value


def ne_certify(cfg: Config, op: int, in_bound: int, operand: int) -> tuple[int, bool]:
    out = C.c_int64()
    st = lib().ne_certify(C.byref(cfg), op, in_bound, operand, C.byref(out))
    if st not in (0, 3):
        raise NeError("ne_certify", st)
    return out.value, st == 0


def ne_gemm_limbs_for(cfg: Config, in_bound: int) -> int:
    return int(lib().ne_gemm_limbs_for(C.byref(cfg), in_bound))


def ne_gemm_limb_plan(cfg: Config, in_bound: int) -> tuple[int, int]:
    """(L, limb_bits): the cheapest exact int8 digit plan of the GEMM operand."""
    b = C.c_int32()
    L = int(lib().ne_gemm_limb_plan(C.byref(cfg), in_bound, C.byref(b)))
    return L, b.value


def diag_new() -> torch.Tensor:
    d = torch.empty(4, dtype=torch.int64, device="cuda")
    ne_diag_reset(d)
    return d


def ne_diag_reset(diag: torch.Tensor) -> None:
    _call("ne_diag_reset", _ptr(diag, torch.int64), _stream())


def diag_read(diag: torch.Tensor) -> dict:
    v = diag.cpu().tolist()
    big = 2 ** 63 - 1
    return {"range_violations": v[0], "first_bad": None if v[1] == big else v[1],
            "fault_positions": v[2], "first_fault": None if v[3] == big else v[3]}


# ------------------------------------------------------------------ a1/a2
def ne_entangle(cfg: Config, c: Sequence[torch.Tensor], eps: Sequence[torch.Tensor], diag=None) -> None:
    n = c[0].numel()
    _call("ne_entangle", C.byref(cfg), _streams(c, torch.int32), n, _streams(eps, torch.int64),
          _ptr(diag, torch.int64), _stream())


def ne_entangle_sets(cfg: Config, c, sets: int, eps, diag=None) -> None:
    """c, eps: sets*M tensors (set s = entries s*M .. s*M+M-1)."""
    _call("ne_entangle_sets", C.byref(cfg), _streams(c, torch.int32), sets, c[0].numel(), _streams(eps, torch.int64),
          _ptr(diag, torch.int64), _stream())


def ne_entangle_sets_w32(cfg: Config, c, sets: int, eps, diag=None) -> None:
    _call("ne_entangle_sets_w32", C.byref(cfg), _streams(c, torch.int32), sets, c[0].numel(),
          _streams(eps, torch.int32), _ptr(diag, torch.int64), _stream())


def ne_entangle_aos(cfg: Config, c, eps_aos: torch.Tensor, diag=None) -> None:
    _call("ne_entangle_aos", C.byref(cfg), _streams(c, torch.int32), c[0].numel(),
          _ptr(eps_aos, torch.int64), _ptr(diag, torch.int64), _stream())


def ne_entangle_limbs(cfg: Config, c, L: int, planes: torch.Tensor, diag=None, limb_bits: int = 8) -> None:
    _call("ne_entangle_limbs", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), L, limb_bits,
          _ptr(planes, torch.int8), _ptr(diag, torch.int64), _stream())


def ne_entangle_stream(cfg: Config, m: int, c_m, c_prev, eps_m, diag=None) -> None:
    _call("ne_entangle_stream", C.byref(cfg), m, _ptr(c_m, torch.int32), _ptr(c_prev, torch.int32),
          _ptr(eps_m, torch.int64), c_m.numel(), _ptr(diag, torch.int64), _stream())


def ne_entangle_limbs_stream(cfg: Config, m: int, c_m, c_prev, L: int, planes_m, diag=None,
                             limb_bits: int = 8) -> None:
    _call("ne_entangle_limbs_stream", C.byref(cfg), m, _ptr(c_m, torch.int32), _ptr(c_prev, torch.int32),
          c_m.numel(), L, limb_bits, _ptr(planes_m, torch.int8), _ptr(diag, torch.int64), _stream())


def ne_op_gemm_limbs_stream(cfg: Config, planes_m, L: int, Bt, rows: int, cols: int, K: int, C_m,
                            limb_bits: int = 8) -> None:
    _call("ne_op_gemm_limbs_stream", C.byref(cfg), _ptr(planes_m, torch.int8), L, limb_bits, _ptr(Bt, torch.int8),
          rows, cols, K, _ptr(C_m, torch.int64), _stream())


def ne_entangle_shared(cfg: Config, g: torch.Tensor, g_ent: torch.Tensor) -> None:
    _call("ne_entangle_shared", C.byref(cfg), _ptr(g, torch.int32), _ptr(g_ent, torch.int64), g.numel(),
          _stream())


# ------------------------------------------------------------------ a3
def ne_op_scale(cfg: Config, x, s: int = 1, g: torch.Tensor | None = None) -> None:
    _call("ne_op_scale", C.byref(cfg), _streams(x, torch.int64), x[0].numel(), int(s), _ptr(g, torch.int32),
          _stream())


def ne_op_add(cfg: Config, x, addend, sign: int = 1) -> None:
    _call("ne_op_add", C.byref(cfg), _streams(x, torch.int64), _streams(addend, torch.int64), x[0].numel(),
          int(sign), _stream())


def ne_op_scale_add(cfg: Config, x, s: int, addend, sign: int = 1, g: torch.Tensor | None = None) -> None:
    _call("ne_op_scale_add", C.byref(cfg), _streams(x, torch.int64), x[0].numel(), int(s), _ptr(g, torch.int32),
          _streams(addend, torch.int64), int(sign), _stream())


def ne_op_inner(cfg: Config, x, v: torch.Tensor, block: int, out) -> None:
    _call("ne_op_inner", C.byref(cfg), _streams(x, torch.int64), x[0].numel(), _ptr(v, torch.int32), v.numel(),
          block, _streams(out, torch.int64), _stream())


def ne_op_outer(cfg: Config, x, h: torch.Tensor, out) -> None:
    _call("ne_op_outer", C.byref(cfg), _streams(x, torch.int64), x[0].numel(), _ptr(h, torch.int32), h.numel(),
          _streams(out, torch.int64), _stream())


def ne_op_conv(cfg: Config, x, g: torch.Tensor, out, correlate: bool = False) -> None:
    _call("ne_op_conv", C.byref(cfg), _streams(x, torch.int64), x[0].numel(), _ptr(g, torch.int32), g.numel(),
          int(correlate), _streams(out, torch.int64), _stream())


def ne_op_permute(cfg: Config, x, perm: torch.Tensor, out) -> None:
    _call("ne_op_permute", C.byref(cfg), _streams(x, torch.int64), _ptr(perm, torch.int32), x[0].numel(),
          _streams(out, torch.int64), _stream())


def ne_gemm_workspace(cfg: Config, rows: int, cols: int, K: int, L: int, LB: int = 1) -> int:
    b = C.c_size_t()
    _call("ne_gemm_workspace", C.byref(cfg), rows, cols, K, L, LB, C.byref(b))
    return b.value


def ne_op_gemm(cfg: Config, A, B: torch.Tensor, rows: int, cols: int, K: int, out, algo: int = NE_GEMM_TC_I8,
               L: int = 4, ws: torch.Tensor | None = None, diag=None, limb_bits: int = 8, LB: int = 1) -> None:
    _call("ne_op_gemm", C.byref(cfg), _streams(A, torch.int64), _ptr(B, torch.int32), rows, cols, K, algo, L, limb_bits,
          LB, _streams(out, torch.int64), _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
          _ptr(diag, torch.int64), _stream())


def ne_op_gemm_plain_i32(planes: torch.Tensor, Bt: torch.Tensor, rows: int, cols: int, K: int, out) -> None:
    """Plain one-digit GEMM with int32 products (the narrowest native baseline)."""
    _call("ne_op_gemm_plain_i32", len(out), _ptr(planes, torch.int8), _ptr(Bt, torch.int8), rows, cols, K,
          _streams(out, torch.int32), _stream())


def ne_gemm_plan_for(cfg: Config, a_bound: int, b_bound: int) -> GemmPlan:
    p = GemmPlan()
    _call("ne_gemm_plan_for", C.byref(cfg), a_bound, b_bound, C.byref(p))
    return p


def ne_entangle_plan(cfg: Config, c, plan: GemmPlan, planes: torch.Tensor, diag=None) -> None:
    _call("ne_entangle_plan", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), C.byref(plan),
          _ptr(planes, torch.int8), _ptr(diag, torch.int64), _stream())


def ne_gemm_prep_b_planes(B: torch.Tensor, K: int, cols: int, LB: int, Bt: torch.Tensor, diag=None) -> None:
    _call("ne_gemm_prep_b_planes", _ptr(B, torch.int32), K, cols, LB, _ptr(Bt, torch.int8), _ptr(diag, torch.int64),
          _stream())


def ne_op_gemm_plan(cfg: Config, planes: torch.Tensor, plan: GemmPlan, Bt: torch.Tensor, rows: int, cols: int,
                    K: int, out) -> None:
    _call("ne_op_gemm_plan", C.byref(cfg), _ptr(planes, torch.int8), C.byref(plan), _ptr(Bt, torch.int8), rows, cols,
          K, _streams(out, torch.int64), _stream())


def ne_gemm_prep_b(B: torch.Tensor, K: int, cols: int, Bt: torch.Tensor, diag=None) -> None:
    _call("ne_gemm_prep_b", _ptr(B, torch.int32), K, cols, _ptr(Bt, torch.int8), _ptr(diag, torch.int64),
          _stream())


def ne_op_gemm_limbs(cfg: Config, planes: torch.Tensor, L: int, Bt: torch.Tensor, rows: int, cols: int, K: int,
                     out, limb_bits: int = 8) -> None:
    _call("ne_op_gemm_limbs", C.byref(cfg), _ptr(planes, torch.int8), L, limb_bits, _ptr(Bt, torch.int8), rows, cols,
          K, _streams(out, torch.int64), _stream())


def ne_op_scale_add_check(cfg: Config, x, s: int, addend, r: int, d_out, bitmap: torch.Tensor | None = None,
                          diag=None, sign: int = 1, g: torch.Tensor | None = None) -> None:
    _call("ne_op_scale_add_check", C.byref(cfg), _streams(x, torch.int64), x[0].numel(), int(s), _ptr(g, torch.int32),
          _streams(addend, torch.int64), int(sign), r, _streams(d_out, torch.int64), _ptr(bitmap, torch.int32),
          _ptr(diag, torch.int64), _stream())


def ne_op_conv_check(cfg: Config, x, g: torch.Tensor, out, r: int, d_out, bitmap: torch.Tensor | None = None,
                     diag=None, correlate: bool = False) -> None:
    _call("ne_op_conv_check", C.byref(cfg), _streams(x, torch.int64), x[0].numel(), _ptr(g, torch.int32), g.numel(),
          int(correlate), _streams(out, torch.int64), r, _streams(d_out, torch.int64), _ptr(bitmap, torch.int32),
          _ptr(diag, torch.int64), _stream())


def ne_op_scale_add_check_w32(cfg: Config, x, s: int, addend, r: int, d_out, bitmap: torch.Tensor | None = None,
                              diag=None, sign: int = 1, g: torch.Tensor | None = None) -> None:
    _call("ne_op_scale_add_check_w32", C.byref(cfg), _streams(x, torch.int32), x[0].numel(), int(s),
          _ptr(g, torch.int32), _streams(addend, torch.int32), int(sign), r, _streams(d_out, torch.int32),
          _ptr(bitmap, torch.int32), _ptr(diag, torch.int64), _stream())


# ------------------------------------------------------------------ w = 32 containers
def ne_entangle_w32(cfg: Config, c, eps, diag=None) -> None:
    _call("ne_entangle_w32", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), _streams(eps, torch.int32),
          _ptr(diag, torch.int64), _stream())


def ne_op_scale_add_w32(cfg: Config, x, s: int = 1, g: torch.Tensor | None = None, addend=None, sign: int = 1) -> None:
    a = C.byref(_streams(addend, torch.int32)) if addend is not None else None
    _call("ne_op_scale_add_w32", C.byref(cfg), _streams(x, torch.int32), x[0].numel(), s, _ptr(g, torch.int32), a,
          sign, _stream())


def ne_disentangle_check_w32(cfg: Config, delta, r: int, d_out, bitmap: torch.Tensor | None = None, diag=None) -> None:
    _call("ne_disentangle_check_w32", C.byref(cfg), _streams(delta, torch.int32), delta[0].numel(), r,
          _streams(d_out, torch.int32), _ptr(bitmap, torch.int32), _ptr(diag, torch.int64), _stream())


def ne_recover_w32(cfg: Config, delta, r: int, d_out) -> None:
    n = next(t for t in delta if t is not None).numel()
    _call("ne_recover_w32", C.byref(cfg), _streams(delta, torch.int32), n, r, _streams(d_out, torch.int32), _stream())


def ne_entangle_aos_w32(cfg: Config, c, x_aos: torch.Tensor, diag=None) -> None:
    """w = 32 AoS containers: x_aos[n*M + m] = eps_m[n] (int32)."""
    _call("ne_entangle_aos_w32", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), _ptr(x_aos, torch.int32),
          _ptr(diag, torch.int64), _stream())


def ne_op_permute_inner_check_w32(cfg: Config, x_aos: torch.Tensor, v: torch.Tensor, block: int, r: int, d_out,
                                  perm: torch.Tensor | None = None, delta_out=None, bitmap: torch.Tensor | None = None,
                                  diag=None) -> None:
    n = x_aos.numel() // cfg.M
    _call("ne_op_permute_inner_check_w32", C.byref(cfg), _ptr(x_aos, torch.int32), _ptr(perm, torch.int32), n,
          _ptr(v, torch.int32), v.numel(), block, r, _streams(delta_out or [], torch.int32),
          _streams(d_out, torch.int32), _ptr(bitmap, torch.int32), _ptr(diag, torch.int64), _stream())


def ne_inject_sweep_w32(cfg: Config, delta, window: int, r: int, flagwords: torch.Tensor, dhat: torch.Tensor) -> None:
    _call("ne_inject_sweep_w32", C.byref(cfg), _streams(delta, torch.int32), window, r, _ptr(flagwords, torch.int64),
          _ptr(dhat, torch.int32), _stream())


def ne_conv_geometry(n: int, taps: int, L: int = 2) -> tuple[int, int, int]:
    """(block, Kpad, plane_len) of the tensor-core convolution."""
    bl, kp, pl = _I32(), _I64(), _I64()
    _call("ne_conv_geometry", n, taps, L, C.byref(bl), C.byref(kp), C.byref(pl))
    return bl.value, kp.value, pl.value


def ne_entangle_limbs_conv(cfg: Config, c, taps: int, correlate: int, L: int, planes: torch.Tensor, diag=None,
                           limb_bits: int = 8, block: int = 128) -> None:
    _call("ne_entangle_limbs_conv", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), taps, correlate, L,
          limb_bits, block, _ptr(planes, torch.int8), _ptr(diag, torch.int64), _stream())


def ne_conv_prep_taps(g: torch.Tensor, correlate: int, Gt: torch.Tensor, diag=None, block: int = 128) -> None:
    _call("ne_conv_prep_taps", _ptr(g, torch.int32), g.numel(), correlate, block, _ptr(Gt, torch.int8),
          _ptr(diag, torch.int64), _stream())


def ne_op_conv_limbs(cfg: Config, planes: torch.Tensor, L: int, Gt: torch.Tensor, n: int, taps: int, correlate: int,
                     out, limb_bits: int = 8, block: int = 128) -> None:
    _call("ne_op_conv_limbs", C.byref(cfg), _ptr(planes, torch.int8), L, limb_bits, block, _ptr(Gt, torch.int8), n,
          taps, correlate, _streams(out, torch.int64), _stream())


def ne_gemm_check_workspace(rows: int, cols: int) -> int:
    b = _SZ()
    _call("ne_gemm_check_workspace", rows, cols, C.byref(b))
    return b.value


def ne_op_gemm_limbs_check(cfg: Config, planes: torch.Tensor, L: int, Bt: torch.Tensor, rows: int, cols: int,
                           K: int, out, r: int, d_out, counters: torch.Tensor, bitmap: torch.Tensor | None = None,
                           diag=None, limb_bits: int = 8) -> None:
    """GEMM + fused disentangle/check epilogue; counters: a zeroed int32 device
    buffer of ne_gemm_check_workspace(rows, cols) bytes (left zeroed)."""
    _call("ne_op_gemm_limbs_check", C.byref(cfg), _ptr(planes, torch.int8), L, limb_bits, _ptr(Bt, torch.int8), rows,
          cols, K, _streams(out, torch.int64), r, _streams(d_out, torch.int64), _ptr(bitmap, torch.int32),
          _ptr(diag, torch.int64), _ptr(counters, torch.int32), _stream())


def ne_op_gemm_limbs_scatter(cfg: Config, planes_m: torch.Tensor, L: int, Bt: torch.Tensor, rows: int, cols: int,
                             K: int, dests, limb_bits: int = 8, local: torch.Tensor | None = None) -> None:
    """One stream's GEMM with output row block j stored into dests[j] (each a
    contiguous int64 device region of rows/len(dests) x cols elements; local
    or peer memory) and, if given, in full into `local`."""
    _call("ne_op_gemm_limbs_scatter", C.byref(cfg), _ptr(planes_m, torch.int8), L, limb_bits, _ptr(Bt, torch.int8),
          rows, cols, K, _streams(dests, torch.int64), len(dests), _ptr(local, torch.int64), _stream())


GEMM_KERNELS = {0: "cta", 1: "pair"}


def ne_gemm_kernel_for(cfg: Config, L: int, limb_bits: int, rows: int, cols: int, K: int) -> str:
    """Which tcgen05 kernel a limb GEMM of this shape/plan launches: "pair" or "cta"."""
    k = _I32()
    _call("ne_gemm_kernel_for", C.byref(cfg), L, limb_bits, rows, cols, K, C.byref(k))
    return GEMM_KERNELS[k.value]


def ne_gemm_trace(buf: torch.Tensor | None, max_clusters: int = 0) -> None:
    """Debug hook: per-CTA tile timestamps of later GEMM launches (see ne.h)."""
    _call("ne_gemm_trace", _ptr(buf, torch.int64), max_clusters)


def ne_gemm_pair_schedule(n_tiles: int, npairs: int) -> int:
    """Pair tiles the CTA-pair kernel keeps whole (the rest run as two halves; see ne.h)."""
    nw = _I64()
    _call("ne_gemm_pair_schedule", n_tiles, npairs, C.byref(nw))
    return nw.value


def ne_gemm_pair_halves(mode: int) -> None:
    """Debug hook: 0 automatic, 1 never halve, 2 halve every pair tile."""
    _call("ne_gemm_pair_halves", mode)


# ------------------------------------------------------------------ a4-a7
def ne_disentangle_check(cfg: Config, delta, r: int, d_out, bitmap: torch.Tensor | None = None, diag=None) -> None:
    _call("ne_disentangle_check", C.byref(cfg), _streams(delta, torch.int64), delta[0].numel(), r,
          _streams(d_out, torch.int64), _ptr(bitmap, torch.int32), _ptr(diag, torch.int64), _stream())


def ne_recover(cfg: Config, delta, r: int, d_out) -> None:
    n = next(t for t in delta if t is not None).numel()
    _call("ne_recover", C.byref(cfg), _streams(delta, torch.int64), n, r, _streams(d_out, torch.int64), _stream())


def ne_op_permute_inner_check(cfg: Config, v: torch.Tensor, block: int, r: int, d_out, *, x=None,
                              x_aos: torch.Tensor | None = None, perm: torch.Tensor | None = None,
                              n: int | None = None, delta_out=None, bitmap=None, diag=None) -> None:
    if n is None:
        n = x_aos.numel() // cfg.M if x_aos is not None else x[0].numel()
    xs = _streams(x if x is not None else [], torch.int64)
    do = _streams(delta_out if delta_out is not None else [], torch.int64)
    _call("ne_op_permute_inner_check", C.byref(cfg), xs, _ptr(x_aos, torch.int64), int(x_aos is not None),
          _ptr(perm, torch.int32), n, _ptr(v, torch.int32), v.numel(), block, r, do, _streams(d_out, torch.int64),
          _ptr(bitmap, torch.int32), _ptr(diag, torch.int64), _stream())


def ne_permute_inner_workspace(cfg: Config, n: int, block: int) -> int:
    """Bytes of device workspace ne_op_permute_inner_check_bucketed needs."""
    b = _SZ()
    _call("ne_permute_inner_workspace", C.byref(cfg), n, block, C.byref(b))
    return b.value


def ne_permute_inner_plan(cfg: Config, n: int, block: int) -> dict:
    """The plan (mode 1 = owned runs, 0 = shared-memory block sums) and geometry
    ne_op_permute_inner_check_bucketed runs for this (M, n, block); host only."""
    mode, S, nwin, nrange = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    rb, cap, ib = C.c_int64(), C.c_int64(), C.c_int64()
    _call("ne_permute_inner_plan", C.byref(cfg), n, block, C.byref(mode), C.byref(S), C.byref(nwin),
          C.byref(nrange), C.byref(rb), C.byref(cap), C.byref(ib))
    return {"mode": mode.value, "S": S.value, "nwin": nwin.value, "nrange": nrange.value, "rb": rb.value,
            "cap": cap.value, "index_bytes": ib.value}


def ne_op_permute_inner_check_bucketed(cfg: Config, x_aos: torch.Tensor, perm: torch.Tensor, v: torch.Tensor,
                                       block: int, r: int, delta, d_out, ws: torch.Tensor, bitmap=None,
                                       diag=None) -> None:
    """The C4 op as a partitioned scatter-reduce (no random gather; see ne.h)."""
    n = x_aos.numel() // cfg.M
    _call("ne_op_permute_inner_check_bucketed", C.byref(cfg), _ptr(x_aos, torch.int64), _ptr(perm, torch.int32), n,
          _ptr(v, torch.int32), v.numel(), block, r, _streams(delta, torch.int64), _streams(d_out, torch.int64),
          _ptr(bitmap, torch.int32), _ptr(diag, torch.int64), _ptr(ws), ws.numel() * ws.element_size(), _stream())


def ne_op_permute_inner_stream(cfg: Config, x_m: torch.Tensor, perm: torch.Tensor, v: torch.Tensor, block: int,
                               b_begin: int, b_count: int, out_m: torch.Tensor) -> None:
    """One stream's gather + blocked inner product over blocks [b_begin, b_begin + b_count)."""
    _call("ne_op_permute_inner_stream", C.byref(cfg), _ptr(x_m, torch.int64), _ptr(perm, torch.int32), x_m.numel(),
          _ptr(v, torch.int32), v.numel(), block, b_begin, b_count, _ptr(out_m, torch.int64), _stream())


# ------------------------------------------------------------------ ABFT comparison baseline (Eqs. 3-6)
def ne_abft_encode_conv(cfg: Config, c, taps: int, correlate: int, block: int, pdata: torch.Tensor, Ls: int,
                        psum: torch.Tensor, diag=None) -> None:
    _call("ne_abft_encode_conv", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), taps, correlate, block,
          _ptr(pdata, torch.int8), Ls, _ptr(psum, torch.int8), _ptr(diag, torch.int64), _stream())


def ne_op_conv_limbs_plain(count: int, planes: torch.Tensor, L: int, Gt: torch.Tensor, n: int, taps: int,
                           correlate: int, out, limb_bits: int = 8, block: int = 128) -> None:
    _call("ne_op_conv_limbs_plain", count, _ptr(planes, torch.int8), L, limb_bits, block, _ptr(Gt, torch.int8), n,
          taps, correlate, _streams(out, torch.int64), _stream())


def ne_abft_encode(cfg: Config, c, r_out: torch.Tensor, diag=None) -> None:
    _call("ne_abft_encode", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), _ptr(r_out, torch.int32),
          _ptr(diag, torch.int64), _stream())


def ne_abft_encode_limbs(cfg: Config, c, pdata: torch.Tensor, Ls: int, psum: torch.Tensor, diag=None) -> None:
    _call("ne_abft_encode_limbs", C.byref(cfg), _streams(c, torch.int32), c[0].numel(), _ptr(pdata, torch.int8), Ls,
          _ptr(psum, torch.int8), _ptr(diag, torch.int64), _stream())


def ne_to_limbs(x, L: int, planes: torch.Tensor, diag=None) -> None:
    _call("ne_to_limbs", _streams(x, torch.int32), len(x), x[0].numel(), L, _ptr(planes, torch.int8),
          _ptr(diag, torch.int64), _stream())


def ne_abft_check(cfg: Config, d, e: torch.Tensor, bitmap=None, diag=None) -> None:
    _call("ne_abft_check", C.byref(cfg), _streams(d, torch.int64), _ptr(e, torch.int64), e.numel(),
          _ptr(bitmap, torch.int32), _ptr(diag, torch.int64), _stream())


def ne_abft_recover(cfg: Config, d, e: torch.Tensor, r: int, d_r: torch.Tensor) -> None:
    _call("ne_abft_recover", C.byref(cfg), _streams(d, torch.int64), _ptr(e, torch.int64), e.numel(), r,
          _ptr(d_r, torch.int64), _stream())


def ne_inject(x: torch.Tensor, idx: int, mask: int) -> None:
    _call("ne_inject", _ptr(x, torch.int64), idx, mask & (2 ** 64 - 1), _stream())


def ne_inject_sweep(cfg: Config, delta, window: int, r: int, flagwords: torch.Tensor, dhat: torch.Tensor) -> None:
    _call("ne_inject_sweep", C.byref(cfg), _streams(delta, torch.int64), window, r, _ptr(flagwords, torch.int64),
          _ptr(dhat, torch.int64), _stream())


# ------------------------------------------------------------------ synthetic inputs (device generator)
def ne_gen_uniform_i32(seed: int, tag: int, gstream: int, lo: int, hi: int, out: torch.Tensor,
                       offset: int = 0) -> None:
    _call("ne_gen_uniform_i32", seed, tag, gstream, lo, hi, offset, out.numel(), _ptr(out, torch.int32), _stream())


def ne_gen_perm_i32(seed: int, tag: int, out: torch.Tensor) -> None:
    _call("ne_gen_perm_i32", seed, tag, out.numel(), _ptr(out, torch.int32), _stream())
