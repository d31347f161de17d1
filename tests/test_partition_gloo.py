"""Multi-process (gloo, CPU) tests of the C1-C4 partitions of SURVEY §8(e)
(paper_1604_04740_b200.dist: part_range, halo_exchange, c4_placement /
c4_payload / c4_allgather) at world 2 and 4 (C4 also 8): every rank computes
its share with the oracle exactly as the GPU ranks do with libne (same
generator offsets, same halo, same gathered layout); the union over ranks is
compared bit-exactly with the oracle run on the whole, unpartitioned problem
and with the plain (unentangled) result."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _c1(O, D, world, rank):
    n, seed = 1000, 0
    ocfg = O.config_for(3, 64)
    lo, hi = D.part_range(n, world, rank, 32)
    c = np.stack([O.gen_uniform(seed, 1, m, -1024, 1024, hi - lo, lo) for m in range(3)])
    a = np.stack([O.gen_uniform(seed, 2, m, -1024, 1024, hi - lo, lo) for m in range(3)])
    delta = O.op_add(ocfg, O.op_scale(ocfg, O.entangle(ocfg, c), 37), O.entangle(ocfg, a))
    d, _, nf = O.disentangle_check(ocfg, delta, 0)
    return lo, hi, delta, d, nf


def _c2(O, D, world, rank):
    n, T, M, seed, H = 4096, 64, 3, 1, D.HALO
    ocfg = O.config_for(M, 64)
    lo, hi = D.part_range(n, world, rank, 32)
    L = hi - lo
    c = np.stack([O.gen_uniform(seed, 1, m, -128, 128, L, lo) for m in range(M)])
    g = O.gen_uniform(seed, 3, 0, -128, 128, T)
    ext = [torch.zeros(H + L, dtype=torch.int64) for _ in range(M)]
    eps = O.entangle(ocfg, c)
    for m in range(M):
        ext[m][H:] = torch.from_numpy(eps[m])
    D.halo_exchange(ext, H, L)
    out = O.op_conv(ocfg, np.stack([t.numpy() for t in ext]), g)[:, H:]
    d, _, nf = O.disentangle_check(ocfg, out, 0)
    return lo, hi, out, d, nf


def _c3(O, D, world, rank):
    M, R, Cc, K, seed = 3, 1024, 64, 64, 2
    ocfg = O.config_for(M, 64)
    r0, r1 = D.part_range(R, world, rank, 256)
    A = np.stack([O.gen_uniform(seed, 4, m, -64, 64, (r1 - r0) * K, r0 * K) for m in range(M)])
    B = O.gen_uniform(seed, 5, 0, -64, 64, K * Cc).reshape(K, Cc)
    delta = O.op_gemm(ocfg, O.entangle(ocfg, A).reshape(M, r1 - r0, K), B).reshape(M, -1)
    d, _, nf = O.disentangle_check(ocfg, delta, 0)
    return r0 * Cc, r1 * Cc, delta, d, nf


def _c4(O, D, world, rank):
    M, n, Bk, seed = 4, 1 << 16, 1024, 3
    ocfg = O.config_for(M, 64)
    nb = n // Bk
    perm = O.gen_perm(seed, 6, n)
    v = O.gen_uniform(seed, 7, 0, -4096, 4096, Bk)
    pieces = []
    for m, lo, hi in D.c4_payload(M, world, rank, nb):
        c = np.zeros((M, n), dtype=np.int64)   # Eq. 15 for stream m needs c_m and c_{m-1} (regenerated)
        c[m] = O.gen_uniform(seed, 1, m, -4096, 4096, n)
        c[(m - 1) % M] = O.gen_uniform(seed, 1, (m - 1) % M, -4096, 4096, n)
        eps_m = O.entangle(ocfg, c)[m]
        pieces.append(torch.from_numpy(O.op_inner(ocfg, eps_m[perm][None, :], v, Bk)[0][lo:hi].copy()))
    full = D.c4_allgather(pieces, M, nb)
    b0, b1 = D.part_range(nb, world, rank, 32)
    delta = np.stack([t[b0:b1].numpy() for t in full])
    d, _, nf = O.disentangle_check(ocfg, delta, 0) if b1 > b0 else (np.zeros((M, 0), np.int64), None, 0)
    full_np = np.stack([t.numpy() for t in full])
    return b0, b1, delta, d, nf, full_np


def _worker(rank, world, port, which, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_1604_04740_b200.dist as D

        out = {}
        for w in which:
            out[w] = {"c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4}[w](O, D, world, rank)
            dist.barrier()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world, which):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, which, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [res[r] for r in range(world)]


def _whole(O, which):
    """The unpartitioned problem through the oracle: (delta, d_hat, plain)."""
    if which == "c1":
        ocfg = O.config_for(3, 64)
        c = np.stack([O.gen_uniform(0, 1, m, -1024, 1024, 1000) for m in range(3)])
        a = np.stack([O.gen_uniform(0, 2, m, -1024, 1024, 1000) for m in range(3)])
        delta = O.op_add(ocfg, O.op_scale(ocfg, O.entangle(ocfg, c), 37), O.entangle(ocfg, a))
        return delta, O.disentangle_check(ocfg, delta, 0)[0], 37 * c + a
    if which == "c2":
        ocfg = O.config_for(3, 64)
        c = np.stack([O.gen_uniform(1, 1, m, -128, 128, 4096) for m in range(3)])
        g = O.gen_uniform(1, 3, 0, -128, 128, 64)
        delta = O.op_conv(ocfg, O.entangle(ocfg, c), g)
        return delta, O.disentangle_check(ocfg, delta, 0)[0], O.op_conv(ocfg, c, g)
    if which == "c3":
        ocfg = O.config_for(3, 64)
        A = np.stack([O.gen_uniform(2, 4, m, -64, 64, 1024 * 64) for m in range(3)]).reshape(3, 1024, 64)
        B = O.gen_uniform(2, 5, 0, -64, 64, 64 * 64).reshape(64, 64)
        delta = O.op_gemm(ocfg, O.entangle(ocfg, A.reshape(3, -1)).reshape(3, 1024, 64), B).reshape(3, -1)
        return delta, O.disentangle_check(ocfg, delta, 0)[0], (A @ B).reshape(3, -1)
    ocfg = O.config_for(4, 64)
    n = 1 << 16
    c = np.stack([O.gen_uniform(3, 1, m, -4096, 4096, n) for m in range(4)])
    perm = O.gen_perm(3, 6, n)
    v = O.gen_uniform(3, 7, 0, -4096, 4096, 1024)
    delta = O.op_inner(ocfg, O.entangle(ocfg, c)[:, perm], v, 1024)
    return delta, O.disentangle_check(ocfg, delta, 0)[0], O.op_inner(ocfg, c[:, perm], v, 1024)


@pytest.mark.parametrize("world", [2, 4])
def test_c1_c2_c3_partitions(O, world):
    res = _run(world, ["c1", "c2", "c3"])
    for which in ("c1", "c2", "c3"):
        delta, d, plain = _whole(O, which)
        cover = 0
        for r in range(world):
            lo, hi, dl, dd, nf = res[r][which]
            assert nf == 0, (which, r)
            assert (dl == delta[:, lo:hi]).all(), (which, r)
            assert (dd == d[:, lo:hi]).all() and (dd == plain[:, lo:hi]).all(), (which, r)
            assert lo == cover, (which, r)   # contiguous, in rank order
            cover = hi
        assert cover == delta.shape[1], which


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_stream_placement(O, world):
    res = _run(world, ["c4"])
    delta, d, plain = _whole(O, "c4")
    cover = 0
    for r in range(world):
        b0, b1, dl, dd, nf, full = res[r]["c4"]
        assert (full == delta).all(), r        # every rank holds all M streams' block sums after the all_gather
        assert nf == 0
        assert (dl == delta[:, b0:b1]).all() and (dd == plain[:, b0:b1]).all(), r
        assert b0 == cover
        cover = b1
    assert cover == delta.shape[1]


def test_placement_geometry():
    import paper_1604_04740_b200.dist as D

    assert D.c4_placement(4, 1, 0) == [(0, 0, 1), (1, 0, 1), (2, 0, 1), (3, 0, 1)]
    assert D.c4_placement(4, 2, 1) == [(1, 0, 1), (3, 0, 1)]
    assert D.c4_placement(4, 8, 5) == [(2, 1, 2)]
    with pytest.raises(ValueError):
        D.c4_placement(4, 6, 0)
    # position ranges tile [0, n) in rank order with aligned interior boundaries
    for n, parts, al in ((4096, 8, 32), (1000, 3, 32), (65536, 8, 32), (4096, 8, 256)):
        rs = [D.part_range(n, parts, j, al) for j in range(parts)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert all(lo % al == 0 for lo, _ in rs)
