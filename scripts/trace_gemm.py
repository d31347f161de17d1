"""Debug: C3 GEMM time and per-tile epilogue (accumulators full -> last chunk
staged) for the current libne.so build."""
import sys

import torch

import paper_1604_04740_b200 as ne

M, R, Cc, K = 3, 4096, 4096, 4096
cfg = ne.ne_config_for(M)
L, b = ne.ne_gemm_limb_plan(cfg, 64)
A = [torch.empty(R * K, dtype=torch.int32, device="cuda") for _ in range(M)]
for m in range(M):
    ne.ne_gen_uniform_i32(2, 4, m, -64, 64, A[m])
B = torch.empty(K * Cc, dtype=torch.int32, device="cuda")
ne.ne_gen_uniform_i32(2, 5, 0, -64, 64, B)
planes = torch.empty(M * L * R * K, dtype=torch.int8, device="cuda")
ne.ne_entangle_limbs(cfg, A, L, planes, limb_bits=b)
Bt = torch.empty(Cc * K, dtype=torch.int8, device="cuda")
ne.ne_gemm_prep_b(B, K, Cc, Bt)
out = [torch.empty(R * Cc, dtype=torch.int64, device="cuda") for _ in range(M)]
ref = [torch.empty(R * Cc, dtype=torch.int64, device="cuda") for _ in range(M)]
tr = torch.zeros(148 * 128, dtype=torch.int64, device="cuda")
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for ncl in (0, 8):
    ne.ne_gemm_trace(tr, ncl)
    tr.zero_()
    ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, b)
    torch.cuda.synchronize()
    ne.ne_gemm_trace(None, ncl)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, b)
    e0.record()
    for _ in range(20):
        ne.ne_op_gemm_limbs(cfg, planes, L, Bt, R, Cc, K, out, b)
    e1.record()
    torch.cuda.synchronize()
    t = tr.view(148, 32, 4).cpu()
    epi, gap, rel, mma, wt = [], [], [], [], []
    for cta in range(148):
        r = [tuple(int(x) for x in row) for row in t[cta].tolist() if row[0] > 0]
        epi += [(e[1] - e[0]) / 1e3 for e in r[1:-1]]
        gap += [(r[i][0] - r[i - 1][0]) / 1e3 for i in range(2, len(r) - 1)]
        rel += [(r[i + 1][2] - r[i][0]) / 1e3 for i in range(1, len(r) - 2)]   # acc full -> next MMA start
        mma += [(r[i][0] - r[i][2]) / 1e3 for i in range(2, len(r) - 1)]       # MMA start -> acc full
        wt += [r[i][3] / 1e3 for i in range(2, len(r) - 1)]                     # MMA waiting on stages
    med = lambda a: sorted(a)[len(a) // 2]
    print(f"{tag} clusters={ncl or 'all'} gemm_ms={e0.elapsed_time(e1) / 20:.4f} item_gap={med(gap):.2f} "
          f"release={med(rel):.2f} mma={med(mma):.2f} (stage waits {med(wt):.2f}) epi_total={med(epi):.2f} us")
ne.ne_gemm_trace(None, 0)
# exactness against the unchanged IMAD64 path on a sample of rows
ws = None
Rs = 256
Es = [torch.empty(Rs * K, dtype=torch.int64, device="cuda") for _ in range(M)]
import oracle as O  # noqa: E402  (debug script: oracle entangle of the sampled rows)
import numpy as np  # noqa: E402
An = np.stack([A[m][:Rs * K].cpu().numpy() for m in range(M)])
E = O.entangle(O.config_for(M, 64), An)
o = [torch.empty(Rs * Cc, dtype=torch.int64, device="cuda") for _ in range(M)]
ne.ne_op_gemm(cfg, [torch.from_numpy(E[m]).cuda() for m in range(M)], B, Rs, Cc, K, o, algo=ne.NE_GEMM_IMAD64)
print(tag, "sample rows exact:", all(torch.equal(o[m], out[m][:Rs * Cc]) for m in range(M)))
