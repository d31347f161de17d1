"""(Runs against commit d1b12b3, the split-K experiment: ne_gemm_pair_split / NE_PAIR_TRACE were reverted after it.)
One C3-shape pair GEMM whole (split 1) then forced split 2, for an ncu capture (experiments)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
import paper_1604_04740_b200 as ne
from split_diag_cases import gemm_case  # noqa: E402

f, out = gemm_case(3, 4096, 4096, 4096)
for s in (1, 2, 0):
    ne.ne_gemm_pair_split(s)
    f()
    torch.cuda.synchronize()
ne.ne_gemm_pair_split(0)
