"""Test-only CPU backend for paper_1604_04740_b200.dist: the same calls as
GpuBackend, computed by the oracle (oracle/), so the multi-process host logic
(stream placement, position-major exchange, survivor routing, checksums) is
exercised over gloo without GPUs.  Never used by the product path."""
import numpy as np
import torch

import oracle as O


class OracleBackend:
    def __init__(self, M: int, bound: int):
        self.cfg = O.config_for(M, 64)
        self.M = M

    def gen(self, seed, tag, stream, lo, hi, n):
        return torch.from_numpy(O.gen_uniform(seed, tag, stream, lo, hi, n))

    def prep_b(self, B, K, cols):
        return B.numpy().reshape(K, cols)

    def entangled_gemm(self, m, A_m, A_prev, Bt, rows, cols, K):
        c = np.zeros((self.M, rows * K), dtype=np.int64)
        c[m] = A_m.numpy()
        c[(m - 1) % self.M] = A_prev.numpy()
        E = O.entangle(self.cfg, c)[m].reshape(rows, K)
        return torch.from_numpy(O.op_gemm(self.cfg, E, Bt).reshape(-1))

    def check(self, deltas, r):
        d, _, nf = O.disentangle_check(self.cfg, np.stack([t.numpy() for t in deltas]), r)
        return [torch.from_numpy(x.copy()) for x in d], nf

    def recover(self, deltas, r):
        d = O.recover(self.cfg, [None if t is None else t.numpy() for t in deltas], r)
        return [torch.from_numpy(x.copy()) for x in d]

    def sync(self):
        pass

    def mark(self, name):
        pass
