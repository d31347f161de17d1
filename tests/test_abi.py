"""C-ABI boundary checks that need no GPU: libne.so loads, exports every
symbol include/*.h declares, and its host-only a0 logic (configuration,
dynamic range, certification, limb count) agrees with the oracle and with
Table II.  No compute calls are made here."""
import ctypes
import os
import re

import pytest

import paper_1604_04740_b200 as ne

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("ne.h", "ne_gendev.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^\s*(?:ne_status|int32_t)\s+(ne_\w+)\s*\(", src, re.M))
    return names


@pytest.fixture(scope="module")
def L():
    ne.build()
    return ne.lib()


def test_every_declared_symbol_is_exported(L):
    declared = _declared()
    assert len(declared) >= 25
    assert declared == set(ne.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_library_is_sm100a(L):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {ne.LIB} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("M", [3, 4, 5, 8, 11, 16, 32])
@pytest.mark.parametrize("w", [32, 64])
def test_config_for_matches_oracle(O, M, w):
    a = ne.ne_config_for(M, w)
    b = O.config_for(M, w)
    assert (a.l, a.k) == (b.l, b.k)


def test_config_errors():
    with pytest.raises(ne.NeError):
        ne.ne_config_for(2, 64)
    with pytest.raises(ne.NeError):
        ne.ne_config_for(33, 64)


@pytest.mark.parametrize("M", [3, 4, 5, 8, 11, 16, 32])
def test_dynamic_range_matches_oracle(O, M):
    assert ne.ne_dynamic_range(ne.ne_config_for(M, 64)) == O.dynamic_range(O.config_for(M, 64))
    assert ne.ne_dynamic_range(ne.ne_config_for(M, 32)) == O.dynamic_range(O.config_for(M, 32))


def test_w32_configs_rejected_by_w64_calls_and_vice_versa():
    """w = 32 containers only through the ne_*_w32 calls, w = 64 only through
    the others (argument validation happens before any device work)."""
    c32, c64 = ne.ne_config_for(3, 32), ne.ne_config_for(3, 64)
    assert (c32.l, c32.k) == (11, 10)
    L = ne.lib()
    st = ne.Streams()
    assert L.ne_entangle(ctypes.byref(c32), st, 0, st, None, None) == 2          # NE_ECONFIG
    assert L.ne_disentangle_check(ctypes.byref(c32), st, 0, 0, st, None, None, None) == 2
    assert L.ne_entangle_w32(ctypes.byref(c64), st, 0, st, None, None) == 2
    assert L.ne_recover_w32(ctypes.byref(c64), st, 0, 0, st, None) == 2
    assert L.ne_disentangle_check_w32(ctypes.byref(c32), st, 0, 3, st, None, None, None) == 4  # NE_EINDEX


def test_certify_baseline_configs():
    c3 = ne.ne_config_for(3)
    b, ok = ne.ne_certify(c3, ne.NE_OP_SCALE, 2 ** 10, 37)
    b, ok2 = ne.ne_certify(c3, ne.NE_OP_ADD, b, 2 ** 10)
    assert b == 38912 and ok and ok2
    assert ne.ne_certify(c3, ne.NE_OP_LINEAR, 128, 64 * 128) == (2 ** 20, True)
    assert ne.ne_certify(c3, ne.NE_OP_LINEAR, 64, 4096 * 64) == (2 ** 24, True)
    c4 = ne.ne_config_for(4)
    assert ne.ne_certify(c4, ne.NE_OP_LINEAR, 2 ** 12, 1024 * 2 ** 12) == (2 ** 34, True)
    hi = ne.ne_dynamic_range(c3)
    assert ne.ne_certify(c3, ne.NE_OP_SCALE, hi, 2)[1] is False


def test_gemm_limbs_for():
    """C3: |E| <= 64 (2^22 + 1) < 2^28 needs 4 balanced int8 digits; C5 (M=8,
    |c| <= 32): |E| <= 8224 needs 2."""
    assert ne.ne_gemm_limbs_for(ne.ne_config_for(3), 64) == 4
    assert ne.ne_gemm_limbs_for(ne.ne_config_for(8), 32) == 2
    assert ne.ne_gemm_limbs_for(ne.ne_config_for(8), 0) == 1


def test_no_cpu_fallback():
    """Compute entry points refuse to run without a CUDA device."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = ne.ne_config_for(3)
    with pytest.raises((RuntimeError, ValueError)):
        ne.ne_op_scale(cfg, [torch.zeros(4, dtype=torch.int64)] * 3, 2)


def test_gemm_limb_plan():
    """Base 2^l, two int8 digits, whenever |c| <= 127 (the digits are then the
    plain halves c_m, c_{m-1} of the entangled value); else base 256."""
    assert ne.ne_gemm_limb_plan(ne.ne_config_for(3), 64) == (2, 22)
    assert ne.ne_gemm_limb_plan(ne.ne_config_for(3), 127) == (2, 22)
    assert ne.ne_gemm_limb_plan(ne.ne_config_for(3), 128) == (4, 8)
    assert ne.ne_gemm_limb_plan(ne.ne_config_for(8), 32) == (2, 8)
    assert ne.ne_gemm_limb_plan(ne.ne_config_for(4), 1000) == (4, 8)


def test_gemm_kernel_for_names_the_timed_kernels():
    """The dispatch query (host-only) names the kernel each launch runs: the
    C3 bench plan (base 2^22, L = 2, 4096^3) runs on the CTA-pair kernel, the
    base-256 plan and short-K / odd shapes on the single-CTA kernel."""
    c3 = ne.ne_config_for(3)
    L, b = ne.ne_gemm_limb_plan(c3, 64)
    assert ne.ne_gemm_kernel_for(c3, L, b, 4096, 4096, 4096) == "pair"
    assert ne.ne_gemm_kernel_for(c3, 4, 8, 4096, 4096, 4096) == "cta"
    assert ne.ne_gemm_kernel_for(c3, L, b, 256, 512, 4096) == "pair"       # smoke()'s pair GEMM
    assert ne.ne_gemm_kernel_for(c3, L, b, 2048, 1280, 2048) == "cta"      # C3P M = 3, N = 2000: 30 pair tiles
    c8 = ne.ne_config_for(8)
    assert ne.ne_gemm_kernel_for(c8, 2, 8, 2048, 16384, 16384) == "cta"    # C5: K > 8192
    assert ne.ne_gemm_kernel_for(c8, 2, 8, 2048, 1024, 2048) == "pair"     # 256 pair tiles at K = 2048
    assert ne.ne_gemm_kernel_for(c3, L, b, 384, 512, 4096) == "cta"        # rows not a multiple of 256
    assert ne.ne_gemm_kernel_for(c3, 1, 8, 4096, 4096, 4096) == "pair"     # one digit: plain baselines, ABFT data
    assert ne.ne_gemm_kernel_for(c3, 1, 8, 512, 512, 4096) == "cta"        # 12 pair tiles: too few
    with pytest.raises(ne.NeError):
        ne.ne_gemm_kernel_for(c3, L, b, 100, 512, 4096)


def test_gemm_plan_for():
    """The digit plan of the wide-range tensor-core GEMM: the two-digit plan
    for |c| <= 127, the split (mixed-radix) plan when 2 x digits(|c|) is
    fewer planes than base-256 digits of eps, else base 256 of eps; B in
    balanced base-256 digits."""
    c3, c4, c8 = ne.ne_config_for(3), ne.ne_config_for(4), ne.ne_config_for(8)

    def plan(cfg, a, b):
        p = ne.ne_gemm_plan_for(cfg, a, b)
        return ("split" if p.kind else "eps", p.LA, p.digit_bits, p.LB, list(p.a_shift)[:p.LA])

    assert plan(c3, 64, 64) == ("eps", 2, 22, 1, [0, 22])
    assert plan(c3, 128, 127) == ("eps", 4, 8, 1, [0, 8, 16, 24])
    assert plan(c3, 1 << 10, 128) == ("split", 4, 8, 2, [0, 8, 22, 30])
    assert plan(c3, 1 << 15, 1 << 15) == ("eps", 5, 8, 3, [0, 8, 16, 24, 32])
    assert plan(c3, 1 << 20, 127) == ("eps", 6, 8, 1, [0, 8, 16, 24, 32, 40])
    assert plan(c8, 32, 32) == ("eps", 2, 8, 1, [0, 8])
    assert plan(c4, 1000, 2 ** 31 - 1)[3] == 5      # every int32 B: 5 balanced digits
    assert plan(c4, 2 ** 31 - 1, 1)[1] <= 8          # every int32 c: at most 8 planes
    with pytest.raises(ne.NeError):
        ne.ne_gemm_plan_for(c3, -1, 1)


def test_argument_validation_of_the_newer_entry_points(L):
    """Errors are returned before any device work (fake, 16-B aligned device
    addresses are never dereferenced): stream-set counts, conv block widths,
    excluded-stream indices, aliasing, geometry arguments."""
    cfg = ne.ne_config_for(3)
    st = ne.Streams()
    fake = [0x10000 * (i + 1) for i in range(8)]
    for i in range(6):
        st.s[i] = fake[i]
    assert L.ne_entangle_sets(ctypes.byref(cfg), st, 11, 16, st, None, None) == 1    # 11 * 3 > 32 streams
    assert L.ne_entangle_sets(ctypes.byref(cfg), st, 0, 16, st, None, None) == 1
    bl, kp, pl = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    assert L.ne_conv_geometry(1000, 4500, 2, ctypes.byref(bl), ctypes.byref(kp), ctypes.byref(pl)) == 0
    assert bl.value == 256 and kp.value % 128 == 0 and kp.value >= 4500 + 255 and pl.value % 256 == 0
    assert L.ne_conv_geometry(1000, 4500, 3, ctypes.byref(bl), ctypes.byref(kp), ctypes.byref(pl)) == 0
    assert bl.value == 128                                                               # 3 limbs: 128-wide
    assert L.ne_conv_geometry(0, 64, 2, ctypes.byref(bl), ctypes.byref(kp), ctypes.byref(pl)) == 1
    assert L.ne_conv_prep_taps(ctypes.c_void_p(fake[0]), 64, 0, 192, ctypes.c_void_p(fake[1]), None, None) == 1
    assert L.ne_op_conv_limbs(ctypes.byref(cfg), ctypes.c_void_p(fake[0]), 3, 8, 256, ctypes.c_void_p(fake[1]),
                              1000, 300, 0, st, None) == 7                              # NE_ENOTSUP: L = 3 at W = 256
    assert L.ne_op_scale_add_check(ctypes.byref(cfg), st, 16, 37, None, st, 1, 3, st, None, None, None) == 4
    assert L.ne_op_conv_check(ctypes.byref(cfg), st, 16, ctypes.c_void_p(fake[7]), 4, 0, st, 0, st, None, None,
                              None) == 1                                                # out aliases x
    assert L.ne_op_gemm_limbs_check(ctypes.byref(cfg), ctypes.c_void_p(fake[0]), 2, 22, ctypes.c_void_p(fake[1]),
                                    128, 128, 128, st, 5, st, None, None, ctypes.c_void_p(fake[2]), None) == 4
    b = ctypes.c_size_t()
    assert L.ne_gemm_check_workspace(256, 512, ctypes.byref(b)) == 0 and b.value >= 2 * 4 * 4
    c32 = ne.ne_config_for(3, 32)
    assert L.ne_op_scale_add_check_w32(ctypes.byref(c32), st, 16, 37, None, st, 1, 3, st, None, None, None) == 4
    assert L.ne_entangle_sets_w32(ctypes.byref(cfg), st, 2, 16, st, None, None) == 2      # w = 64 config
    # fused GEMM -> exchange: destination count, alignment, row blocks of whole tiles
    P = ctypes.c_void_p
    assert L.ne_op_gemm_limbs_scatter(ctypes.byref(cfg), P(fake[0]), 2, 22, P(fake[1]), 1024, 256, 256, st, 0,
                                      None, None) == 1                                  # ndest = 0
    assert L.ne_op_gemm_limbs_scatter(ctypes.byref(cfg), P(fake[0]), 2, 22, P(fake[1]), 1024, 256, 256, st, 9,
                                      None, None) == 1                                  # ndest > 8
    assert L.ne_op_gemm_limbs_scatter(ctypes.byref(cfg), P(fake[0]), 2, 22, P(fake[1]), 1024, 256, 256, st, 7,
                                      None, None) == 1                                  # dests[6] is NULL
    assert L.ne_op_gemm_limbs_scatter(ctypes.byref(cfg), P(fake[0]), 2, 22, P(fake[1]), 1024, 256, 256, st, 2,
                                      P(fake[2] + 8), None) == 1                        # misaligned local copy
    assert L.ne_op_gemm_limbs_scatter(ctypes.byref(cfg), P(fake[0]), 2, 22, P(fake[1]), 384, 256, 256, st, 2,
                                      None, None) == 7                                  # 192-row blocks: ENOTSUP
    assert L.ne_gemm_trace(None, -1) == 1
    assert L.ne_gemm_trace(None, 0) == 0


def test_sass_has_tcgen05_tma_and_tmem(L):
    """The GEMM / conv kernels are real tcgen05 code: the sm_100a SASS of
    libne.so contains the tensor-core MMA (UTCIMMA), its commit barrier
    (UTCBAR), TMEM allocation (UTCATOMSWS) and loads (LDTM), and TMA bulk
    tensor loads / stores (UTMALDG / UTMASTG)."""
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {ne.LIB} 2>/dev/null").read()
    for op in ("UTCIMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "UTMALDG", "UTMASTG"):
        assert op in sass, op


def test_empty_inputs_are_no_ops(L):
    """n_total = 0 is a valid, empty problem for every streaming entry point:
    NE_OK before any pointer is inspected or any kernel is enqueued (no device
    is needed, NULL buffers are fine)."""
    c64, c32 = ne.ne_config_for(3), ne.ne_config_for(3, 32)
    S = ne.Streams()        # all NULL
    N = None
    B = ctypes.byref
    calls = {
        "ne_entangle": (B(c64), S, 0, S, N, N),
        "ne_entangle_sets": (B(c64), S, 2, 0, S, N, N),
        "ne_entangle_aos": (B(c64), S, 0, N, N, N),
        "ne_entangle_w32": (B(c32), S, 0, S, N, N),
        "ne_entangle_aos_w32": (B(c32), S, 0, N, N, N),
        "ne_op_scale": (B(c64), S, 0, 3, N, N),
        "ne_op_add": (B(c64), S, S, 0, 1, N),
        "ne_op_scale_add": (B(c64), S, 0, 3, N, S, 1, N),
        "ne_op_scale_add_w32": (B(c32), S, 0, 3, N, N, 1, N),
        "ne_disentangle_check": (B(c64), S, 0, 0, S, N, N, N),
        "ne_disentangle_check_w32": (B(c32), S, 0, 0, S, N, N, N),
        "ne_op_permute": (B(c64), S, N, 0, S, N),
        "ne_op_inner": (B(c64), S, 0, N, 1, 1, S, N),
        "ne_op_permute_inner_check": (B(c64), S, N, 1, N, 0, N, 1, 1, 0, S, S, N, N, N),
        "ne_op_permute_inner_check_w32": (B(c32), N, N, 0, N, 1, 1, 0, S, S, N, N, N),
        "ne_entangle_shared": (B(c64), N, N, 0, N),
    }
    for name, args in calls.items():
        assert getattr(L, name)(*args) == 0, name


def test_gemm_pair_schedule(L):
    """The CTA-pair kernel keeps whole tiles except a last partial wave of r
    tiles with 2 r <= pairs, which runs as 2 r half tiles: C3's 768 tiles on
    74 pairs -> 740 whole + 28 halved; the paper's M = 8, N = 2000 GEMM (320
    tiles) -> 296 whole; 48 or 128 tiles (r = 48 / 54 > 37) stay whole; full
    waves stay whole; 12 tiles on 74 pairs are all halved."""
    assert ne.ne_gemm_pair_schedule(768, 74) == 740
    assert ne.ne_gemm_pair_schedule(320, 74) == 296
    assert ne.ne_gemm_pair_schedule(48, 74) == 48
    assert ne.ne_gemm_pair_schedule(128, 74) == 128
    assert ne.ne_gemm_pair_schedule(740, 74) == 740
    assert ne.ne_gemm_pair_schedule(12, 74) == 0
    assert ne.ne_gemm_pair_schedule(0, 74) == 0
    with pytest.raises(ne.NeError):
        ne.ne_gemm_pair_schedule(10, 0)
    with pytest.raises(ne.NeError):
        ne.ne_gemm_pair_halves(3)


def test_permute_inner_plan():
    """ne_permute_inner_plan (host only): the C4 config (M = 4, n = 2^28,
    blocks of 1024) runs the owned-run mode with 64 MB windows and one reduce
    CTA per SM; blocks that do not tile the 4096-position scatter chunk take
    the shared-atomic mode; the workspace holds the 32-bit pairs, the run
    index and the overflow list."""
    cfg = ne.ne_config_for(4)
    p = ne.ne_permute_inner_plan(cfg, 1 << 28, 1024)
    assert p["mode"] == 1 and p["S"] == 21 and p["nwin"] == 128
    assert p["nrange"] <= 148 and p["rb"] % 4 == 0 and p["rb"] * p["nrange"] >= (1 << 18)
    cells = p["nwin"] * p["nrange"]
    assert p["index_bytes"] == cells * p["rb"] * 4
    assert cells * p["cap"] >= 1 << 28 and p["cap"] < 65536
    ws = ne.ne_permute_inner_workspace(cfg, 1 << 28, 1024)
    assert ws >= cells * p["cap"] * 4 + p["index_bytes"] + (1 << 28) * 8
    for M, n, B in [(4, 100003, 100), (5, 4099, 7), (4, 1 << 20, 3000)]:
        q = ne.ne_permute_inner_plan(ne.ne_config_for(M), n, B)
        assert q["mode"] == 0 and q["index_bytes"] == 0
    for M, n, B in [(8, 65536, 1024), (4, 70000, 4096), (3, 1, 1024), (8, 1 << 28, 1024)]:
        assert ne.ne_permute_inner_plan(ne.ne_config_for(M), n, B)["mode"] == 1
    assert ne.ne_permute_inner_plan(ne.ne_config_for(8), 1 << 28, 1024)["nrange"] <= 148
    for n, B in [(-1, 1024), (1 << 31, 1024), (10, 0)]:
        with pytest.raises(ne.NeError):
            ne.ne_permute_inner_plan(cfg, n, B)
