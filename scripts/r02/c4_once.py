"""One C4 permute + inner + check stage (partitioned form) after a warm-up: for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1604_04740_b200 as ne
M, n, B = 4, 1 << 28, 1024
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
ws = torch.empty(ne.ne_permute_inner_workspace(cfg, n, B), dtype=torch.uint8, device='cuda')
for _ in range(int(os.environ.get("REPS", "2"))):
    ne.ne_op_permute_inner_check_bucketed(cfg, eps, perm, v, B, 0, delta, dout, ws)
torch.cuda.synchronize()
print("ok")
