"""Experiment: effect of cudaLimitMaxL2FetchGranularity on the C4 random gather."""
import ctypes
import glob
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_04740_b200 as ne  # noqa: E402

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
cands += ["/usr/local/cuda/lib64/libcudart.so"]
rt = None
for c in cands:
    try:
        rt = ctypes.CDLL(c)
        break
    except OSError:
        pass
LIM = 0x05  # cudaLimitMaxL2FetchGranularity


def get():
    v = ctypes.c_size_t()
    rt.cudaDeviceGetLimit(ctypes.byref(v), LIM)
    return v.value


n = 1 << 28 if len(sys.argv) < 2 else int(sys.argv[1])
cfg = ne.ne_config_for(4)
c = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(4)]
for m in range(4):
    ne.ne_gen_uniform_i32(3, 1, m, -4096, 4096, c[m])
perm = torch.empty(n, dtype=torch.int32, device="cuda")
ne.ne_gen_perm_i32(3, 6, perm)
v = torch.empty(1024, dtype=torch.int32, device="cuda")
ne.ne_gen_uniform_i32(3, 7, 0, -4096, 4096, v)
eps = torch.empty(4 * n, dtype=torch.int64, device="cuda")
ne.ne_entangle_aos(cfg, c, eps)
nb = n // 1024
d = [torch.empty(nb, dtype=torch.int64, device="cuda") for _ in range(4)]
print("default limit", get())
for g in (get(), 128, 64, 32, 0):
    st = rt.cudaDeviceSetLimit(LIM, ctypes.c_size_t(g))
    for _ in range(2):
        ne.ne_op_permute_inner_check(cfg, v, 1024, 0, d, x_aos=eps, perm=perm, n=n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        ne.ne_op_permute_inner_check(cfg, v, 1024, 0, d, x_aos=eps, perm=perm, n=n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"set {g} (rc {st}) -> limit {get()}: {ms:.3f} ms, algorithmic {n * 36 / ms / 1e6:.0f} GB/s")
