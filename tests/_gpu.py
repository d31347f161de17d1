"""Helpers for the GPU parity tests: move seeded numpy inputs to separately
allocated (hence 16-byte aligned) CUDA streams and back."""
import numpy as np
import torch


def to_streams(a, dtype=torch.int32):
    """(M, N) numpy -> list of M contiguous CUDA tensors (one allocation each)."""
    return [torch.from_numpy(np.ascontiguousarray(row)).to(dtype).cuda() for row in np.asarray(a)]


def empty_streams(M, N, dtype=torch.int64):
    return [torch.empty(N, dtype=dtype, device="cuda") for _ in range(M)]


def to_np(streams):
    return np.stack([t.cpu().numpy().astype(np.int64) for t in streams])


def dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dtype).cuda()


def bitmap_to_flags(bm, n):
    w = bm.cpu().numpy().astype(np.uint32)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")
    return bits[:n].astype(np.uint8)


def flags_to_bitmap(flags):
    n = len(flags)
    nw = (n + 31) // 32
    padded = np.zeros(nw * 32, dtype=np.uint8)
    padded[:n] = flags
    return np.packbits(padded, bitorder="little").view(np.uint32)
