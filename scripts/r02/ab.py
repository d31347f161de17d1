"""A/B timing of libne build variants on one box (experiments only).

    python scripts/r02/ab.py --variant old:-DNE_CONV_ENTANGLE_OLD --variant new: --case conv_entangle
    python scripts/r02/ab.py --variant base@HEAD: --variant new: --case c3_gemm   # after
        git archive HEAD paper_1604_04740_b200/csrc include gen | tar -x -C .ab_src/HEAD  (here, before gpurun)

Each variant is compiled (the _build flags + its -D flags) into
/tmp/ne_ab/<name>/libne.so; each case is then timed in a fresh process per
variant with CUDA events (median of reps), alternating variants 3 times."""
import argparse
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def build(name, flags):
    import paper_1604_04740_b200._build as B

    out = f"/tmp/ne_ab/{name}"
    os.makedirs(out, exist_ok=True)
    objs = []
    procs = []
    csrc, inc = B.CSRC, []
    if "@" in name:  # sources of another revision, exported under .ab_src/<rev>
        tree = os.path.join(ROOT, ".ab_src", name.split("@", 1)[1])
        csrc, inc = os.path.join(tree, "paper_1604_04740_b200", "csrc"), ["-I", os.path.join(tree, "include")]
    for src in sorted(glob.glob(os.path.join(csrc, "*.cu"))):
        obj = os.path.join(out, os.path.basename(src) + ".o")
        procs.append(subprocess.Popen([B.NVCC, *B.ARCH, *inc, *B.FLAGS, *flags, "-c", src, "-o", obj]))
        objs.append(obj)
    assert all(p.wait() == 0 for p in procs)
    lib = os.path.join(out, "libne.so")
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs])
    return lib


CASES = {
    "conv_entangle": """
M, N, T = {M}, 10 ** 6, {T}
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 127)
bw, kp, plen = ne.ne_conv_geometry(N, T, L)
c = [torch.randint(-128, 128, (N,), dtype=torch.int32, device='cuda') for _ in range(M)]
planes = torch.empty(M * L * plen, dtype=torch.int8, device='cuda')
f = lambda: ne.ne_entangle_limbs_conv(cfg, c, T, 0, L, planes, None, b, bw)
""",
    "conv_gemm": """
M, N, T = {M}, 10 ** 6, {T}
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 127)
bw, kp, plen = ne.ne_conv_geometry(N, T, L)
c = [torch.randint(-128, 128, (N,), dtype=torch.int32, device='cuda') for _ in range(M)]
planes = torch.empty(M * L * plen, dtype=torch.int8, device='cuda')
g = torch.randint(-128, 128, (T,), dtype=torch.int32, device='cuda')
Gt = torch.empty(bw * kp, dtype=torch.int8, device='cuda')
ne.ne_entangle_limbs_conv(cfg, c, T, 0, L, planes, None, b, bw)
ne.ne_conv_prep_taps(g, 0, Gt, None, bw)
out = [torch.empty(N, dtype=torch.int64, device='cuda') for _ in range(M)]
f = lambda: ne.ne_op_conv_limbs(cfg, planes, L, Gt, N, T, 0, out, b, bw)
""",
    "conv_gemm128": """
M, N, T = {M}, 10 ** 6, {T}   # the paper's conv shape with 128-output blocks forced (single-CTA 128 x 128 tiles)
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 127)
bw = 128
kp = (T + bw - 1 + 127) // 128 * 128
plen = (bw * ((N + bw - 1) // bw) + kp + bw - 1) // bw * bw
c = [torch.randint(-128, 128, (N,), dtype=torch.int32, device='cuda') for _ in range(M)]
planes = torch.empty(M * L * plen, dtype=torch.int8, device='cuda')
taps = torch.randint(-128, 128, (T,), dtype=torch.int32, device='cuda')
Gt = torch.empty(bw * kp, dtype=torch.int8, device='cuda')
ne.ne_entangle_limbs_conv(cfg, c, T, 0, L, planes, None, b, bw)
ne.ne_conv_prep_taps(taps, 0, Gt, None, bw)
out = [torch.empty(N, dtype=torch.int64, device='cuda') for _ in range(M)]
f = lambda: ne.ne_op_conv_limbs(cfg, planes, L, Gt, N, T, 0, out, b, bw)
""",
    "c4_permute": """
M, n, B = 4, 1 << 28, 1024   # C4's permute + inner + check stage (--T 1: the partitioned scatter-reduce)
cfg = ne.ne_config_for(M)
c = [torch.randint(-4096, 4096, (n,), dtype=torch.int32, device='cuda') for _ in range(M)]
eps = torch.empty(n * M, dtype=torch.int64, device='cuda')
ne.ne_entangle_aos(cfg, c, eps)
del c
perm = torch.empty(n, dtype=torch.int32, device='cuda')
ne.ne_gen_perm_i32(3, 6, perm)
v = torch.randint(-4096, 4096, (B,), dtype=torch.int32, device='cuda')
nb = n // B
delta = [torch.empty(nb, dtype=torch.int64, device='cuda') for _ in range(M)]
dout = [torch.empty(nb, dtype=torch.int64, device='cuda') for _ in range(M)]
if {T} == 1:
    ws = torch.empty(ne.ne_permute_inner_workspace(cfg, n, B), dtype=torch.uint8, device='cuda')
    f = lambda: ne.ne_op_permute_inner_check_bucketed(cfg, eps, perm, v, B, 0, delta, dout, ws)
else:
    f = lambda: ne.ne_op_permute_inner_check(cfg, v, B, 0, dout, x_aos=eps, perm=perm, n=n, delta_out=delta)
""",
    "c1_sac": """
M, n = 3, 1 << 27
cfg = ne.ne_config_for(M)
c = [torch.randint(-1024, 1024, (n,), dtype=torch.int32, device='cuda') for _ in range(2 * M)]
eps = [torch.empty(n, dtype=torch.int64, device='cuda') for _ in range(2 * M)]
ne.ne_entangle_sets(cfg, c, 2, eps)
d = [torch.empty(n, dtype=torch.int64, device='cuda') for _ in range(M)]
bm = torch.empty(n // 32, dtype=torch.int32, device='cuda')
f = lambda: ne.ne_op_scale_add_check(cfg, eps[:M], 1, eps[M:], 0, d, bm)
""",
    "c3_gemm_rank8": """
M, n, R = 3, 4096, 512   # C3's row split at N = 8: 96 pair tiles (split-K 2 by the heuristic)
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 64)
A = [torch.randint(-64, 64, (R * n,), dtype=torch.int32, device='cuda') for _ in range(M)]
planes = torch.empty(M * L * R * n, dtype=torch.int8, device='cuda')
ne.ne_entangle_limbs(cfg, A, L, planes, None, b)
Bt = torch.randint(-64, 64, (n * n,), dtype=torch.int8, device='cuda')
out = [torch.empty(R * n, dtype=torch.int64, device='cuda') for _ in range(M)]
f = lambda: ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, n, n, out, b)
""",
    "c3p_gemm": """
M, R, Cc, K = {M}, 2048, 1280, {T}   # the paper's GEMM shape, padded (rows 2000 -> 2048, cols 1200 -> 1280)
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 64)
A = [torch.randint(-64, 64, (R * K,), dtype=torch.int32, device='cuda') for _ in range(M)]
planes = torch.empty(M * L * R * K, dtype=torch.int8, device='cuda')
ne.ne_entangle_limbs(cfg, A, L, planes, None, b)
Bt = torch.randint(-64, 64, (Cc * K,), dtype=torch.int8, device='cuda')
out = [torch.empty(R * Cc, dtype=torch.int64, device='cuda') for _ in range(M)]
f = lambda: ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, b)
""",
    "c2_conv_check": """
M, N, T = {M}, 65536, {T}   # C2: 3 x 65536 outputs, 64 taps (--M 3 --T 64)
cfg = ne.ne_config_for(M)
c = [torch.randint(-128, 128, (N,), dtype=torch.int32, device='cuda') for _ in range(M)]
eps = [torch.empty(N, dtype=torch.int64, device='cuda') for _ in range(M)]
ne.ne_entangle(cfg, c, eps)
taps = torch.randint(-128, 128, (T,), dtype=torch.int32, device='cuda')
out = [torch.empty(N, dtype=torch.int64, device='cuda') for _ in range(M)]
d = [torch.empty(N, dtype=torch.int64, device='cuda') for _ in range(M)]
f = lambda: ne.ne_op_conv_check(cfg, eps, taps, out, 0, d)
""",
    "c3_entangle": """
M, n = 3, 4096   # C3's operand: 3 x 4096^2 int32 -> two base-2^22 digit planes per stream
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 64)
A = [torch.randint(-64, 64, (n * n,), dtype=torch.int32, device='cuda') for _ in range(M)]
planes = torch.empty(M * L * n * n, dtype=torch.int8, device='cuda')
f = lambda: ne.ne_entangle_limbs(cfg, A, L, planes, None, b)
""",
    "prep_b": """
K, C = 4096, 4096   # C3's B operand: int32 K x cols -> int8 cols x K
B = torch.randint(-128, 128, (K * C,), dtype=torch.int32, device='cuda')
Bt = torch.empty(C * K, dtype=torch.int8, device='cuda')
f = lambda: ne.ne_gemm_prep_b(B, K, C, Bt)
""",
    "c3_gemm": """
M, n = 3, 4096
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 64)
A = [torch.randint(-64, 64, (n * n,), dtype=torch.int32, device='cuda') for _ in range(M)]
planes = torch.empty(M * L * n * n, dtype=torch.int8, device='cuda')
ne.ne_entangle_limbs(cfg, A, L, planes, None, b)
Bt = torch.randint(-64, 64, (n * n,), dtype=torch.int8, device='cuda')
out = [torch.empty(n * n, dtype=torch.int64, device='cuda') for _ in range(M)]
f = lambda: ne.ne_op_gemm_limbs(cfg, planes, L, Bt, n, n, n, out, b)
""",
}

TIMER = """
import sys, statistics, torch
sys.path.insert(0, {root!r})
import ctypes
import paper_1604_04740_b200 as ne
ne.LIB = {lib!r}
_L = ctypes.CDLL(ne.LIB)
ne._SIGS = {{k: v for k, v in ne._SIGS.items() if hasattr(_L, k)}}  # an older build lacks newer calls
ne.lib()
{pre}
{setup}
for _ in range(5): f()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    f()
ts = []
flush = torch.empty(1 << 29, dtype=torch.uint8, device='cuda') if {flush} else None
for _ in range({reps}):
    if flush is not None:
        flush.fill_(1)   # 512 MB: L2 cold for the replay (outside the events)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(statistics.median(ts))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", action="append", required=True, help="name:flags (space separated)")
    ap.add_argument("--case", required=True)
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--T", type=int, default=4500)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--flush", action="store_true", help="flush L2 (512 MB write) before every replay")
    ap.add_argument("--pre", default="", help="python run after loading (e.g. ne.ne_gemm_pair_split(1))")
    a = ap.parse_args()
    libs, pres, built = {}, {}, {}
    for v in a.variant:
        name, flags = v.split(":", 1)
        toks = flags.split()
        cflags = [t for t in toks if not t.startswith("py:")]
        pres[name] = "\n".join(t[3:] for t in toks if t.startswith("py:"))  # e.g. py:ne.ne_gemm_pair_split(1)
        key = (name.split("@", 1)[1] if "@" in name else "", tuple(cflags))
        if key not in built:
            built[key] = build(name, cflags)
        libs[name] = built[key]
    setup = CASES[a.case].format(M=a.M, T=a.T)
    res = {k: [] for k in libs}
    for _ in range(3):
        for name, lib in libs.items():
            code = TIMER.format(root=ROOT, lib=lib, setup=setup, reps=a.reps, flush=a.flush, pre="\n".join(x for x in (a.pre if "@" not in name else "", pres[name]) if x))
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
            if r.returncode:
                print(name, "failed:", r.stderr[-2000:])
                continue
            res[name].append(float(r.stdout.strip().splitlines()[-1]))
    for name, v in res.items():
        print(f"{a.case} M={a.M} T={a.T} {name}: " + " ".join(f"{x * 1e3:.1f}" for x in v) + " us")


if __name__ == "__main__":
    main()
