"""(Runs against commit d1b12b3, the split-K experiment: ne_gemm_pair_split / NE_PAIR_TRACE were reverted after it.)
Split-K diagnostics (experiments): eager vs graph-replayed timing of the
pair-kernel conv / GEMM under forced split factors."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
import paper_1604_04740_b200 as ne


from split_diag_cases import conv_case, gemm_case  # noqa: E402


def eager(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def graph(f, reps=20):
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


cases = {"conv M=3 T=4500": lambda: conv_case(3, 4500), "conv M=8 T=4500": lambda: conv_case(8, 4500),
         "c3 gemm": lambda: gemm_case(3, 4096, 4096, 4096), "c3p M=8": lambda: gemm_case(8, 2048, 1280, 2048)}
for name, mk in cases.items():
    f, out = mk()
    ref = None
    for s in (1, 0, 2, 3, 4):
        ne.ne_gemm_pair_split(s)
        te = eager(f)
        tg = graph(f)
        same = None
        if ref is None:
            ref = [o.clone() for o in out]
        else:
            same = all(torch.equal(o, r) for o, r in zip(out, ref))
        print(f"{name} split={s}: eager {te:.1f} us  graph {tg:.1f} us  equal={same}", flush=True)
    ne.ne_gemm_pair_split(0)
