"""(Runs against commit d1b12b3, the split-K experiment: ne_gemm_pair_split / NE_PAIR_TRACE were reverted after it.)
Per-item timeline of the CTA-pair kernel (experiments): builds libne with
-DNE_PAIR_TRACE, runs one C3-shape GEMM under a given split setting and prints
the last rounds' items (MMA pass starts, limb-0 complete, after the chain
wait, epilogue end; microseconds from the first MMA start)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
import ab  # noqa: E402
import paper_1604_04740_b200 as ne  # noqa: E402

lib = ab.build("trace", ["-DNE_PAIR_TRACE"])
ne.LIB = lib
ne.lib()
L = ctypes.CDLL(lib)
L.ne_dbg_pair_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
from split_diag_cases import conv_case, gemm_case  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c3"
split = int(sys.argv[2]) if len(sys.argv) > 2 else 0
f, _ = gemm_case(3, 4096, 4096, 4096) if case == "c3" else conv_case(3, 4500)
ne.ne_gemm_pair_split(split)
for _ in range(3):
    f()
torch.cuda.synchronize()
L.ne_dbg_pair_trace(None, 1)
f()
torch.cuda.synchronize()
buf = np.zeros(160 * 32 * 8, dtype=np.int64)
L.ne_dbg_pair_trace(buf.ctypes.data, 0)
t = buf.reshape(160, 32, 8)
lead = t[0::2]                       # leader CTAs: MMA pass starts in [1], [2]
t0 = lead[:, :, 1][lead[:, :, 1] > 0].min()
us = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")
print(f"case {case} split {split}")
ends = []
for p in range(lead.shape[0]):
    items = [(int(lead[p, i, 0]), us(lead[p, i, 1]), us(lead[p, i, 2]), us(lead[p, i, 3]), us(lead[p, i, 4]),
              us(lead[p, i, 5])) for i in range(32) if lead[p, i, 1] > 0]
    if not items:
        continue
    ends.append(max(x[3] for x in items))
    if p % 8 == 0 or p >= 54:
        print(f"pair {p}: " + " | ".join(f"w{w} m{a:.1f}/{b:.1f} f{c:.1f} r{d:.1f} e{e:.1f}" for w, a, b, c, d, e in items[-3:]))
print("last limb-0 complete per pair: max %.1f  min %.1f" % (np.nanmax(ends), np.nanmin(ends)))
ne.ne_gemm_pair_split(0)
