"""Test-only CPU backend for paper_1604_04740_b200.dist: the same calls as
GpuBackend, computed by the oracle (oracle/), so the multi-process host logic
(stream placement, position-major exchange, survivor routing, checksums) is
exercised over gloo without GPUs.  Never used by the product path."""
import numpy as np
import torch
import torch.distributed as dist

import oracle as O


class _Slot:
    """Placeholder for a slice of rank j's window (the CPU emulation has no
    peer memory): stores into it are recorded and delivered at barrier()."""

    def __init__(self, win, j, lo, hi):
        self.win, self.j, self.lo, self.hi = win, j, lo, hi

    def __getitem__(self, sl):
        assert sl.step is None
        return _Slot(self.win, self.j, self.lo + sl.start, self.lo + sl.stop)


class EmulatedWindow:
    """gloo emulation of dist.SymmWindow: peer(j)[a:b] is a store target in
    rank j's window; barrier() delivers every rank's recorded stores."""

    def __init__(self, n):
        self.local = torch.zeros(n, dtype=torch.int64)
        self.pending = []

    def peer(self, j):
        return _Slot(self, j, 0, self.local.numel())

    def store(self, slot, data):
        assert data.numel() == slot.hi - slot.lo
        self.pending.append((slot.j, slot.lo, data.clone()))

    def barrier(self):
        world = dist.get_world_size() if dist.is_initialized() else 1
        me = dist.get_rank() if dist.is_initialized() else 0
        allp = [None] * world
        if world > 1:
            dist.all_gather_object(allp, self.pending)
        else:
            allp = [self.pending]
        for sent in allp:
            for j, lo, data in sent:
                if j == me:
                    self.local[lo:lo + data.numel()] = data
        self.pending = []


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

    def exchange_window(self, n):
        return EmulatedWindow(n)

    def entangled_gemm_scatter(self, m, A_m, A_prev, Bt, rows, cols, K, dests, keep_local):
        """Row block j of Delta_m goes to dests[j] (what the fused kernel
        stores over NVLink), recorded here and delivered at the barrier."""
        d = self.entangled_gemm(m, A_m, A_prev, Bt, rows, cols, K)
        nd = len(dests)
        blk = rows // nd * cols
        for j, slot in enumerate(dests):
            slot.win.store(slot, d[j * blk:(j + 1) * blk])
        return d if keep_local else None

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
