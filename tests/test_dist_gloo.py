"""Multi-process (gloo, CPU) tests of the C5 orchestration in
paper_1604_04740_b200.dist: one entangled stream per rank (world = M = 8) and
several streams per rank (world = 2), position-major exchange, the
reliability check on every rank's slice, a simulated fail-stop of one stream /
rank and recovery by the survivors.  Compute is the oracle (test backend);
expected values are the plain integer products computed here with numpy."""
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


def _worker(rank, world, port, plans, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from _oracle_backend import OracleBackend
        from paper_1604_04740_b200.dist import C5Plan, c5_run, make_survivor_groups

        results = []
        groups_for = {}
        for plan_kw in plans:
            plan = C5Plan(**plan_kw)
            if plan.M not in groups_for:
                groups_for[plan.M] = make_survivor_groups(world, plan.M)
            res = c5_run(OracleBackend(plan.M, plan.bound), plan, groups_for[plan.M])
            # expected: plain products A_m B (no entanglement), from the same generator
            M, R, Cc, K, b = plan.M, plan.rows, plan.cols, plan.K, plan.bound
            B = O.gen_uniform(plan.seed, 5, 0, -b, b, K * Cc).reshape(K, Cc)
            plain = np.stack([(O.gen_uniform(plan.seed, 4, m, -b, b, R * K).reshape(R, K) @ B).reshape(-1)
                              for m in range(M)])
            lo, d = res["check_slice"]
            ok_check = all((d[m].numpy() == plain[m, lo:lo + d[m].numel()]).all() for m in range(M))
            ok_rec = None
            if "recover_slice" in res:
                lo2, d2 = res["recover_slice"]
                ok_rec = all((d2[m].numpy() == plain[m, lo2:lo2 + d2[m].numel()]).all() for m in range(M))
            results.append((rank, res["flagged"], res.get("checksum_ok"), ok_check, ok_rec, res["streams"]))
            dist.barrier()
        q.put(results)
    finally:
        dist.destroy_process_group()


def _run(world, plans):
    """Run every plan in one set of `world` spawned gloo processes; returns,
    per plan, the sorted per-rank results."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, plans, q)) for r in range(world)]
    for p in procs:
        p.start()
    per_rank = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [sorted(rk[i] for rk in per_rank) for i in range(len(plans))]


SMALL = dict(M=8, rows_total=32, cols=8, K=16, seed=4, bound=32)
W2_PLANS = [dict(SMALL, kill=0), dict(SMALL, kill=5), dict(SMALL, kill=None),
            dict(M=3, rows_total=45, cols=7, K=5, seed=9, bound=32, kill=1)]


@pytest.fixture(scope="module")
def world2():
    return _run(2, W2_PLANS)


def test_c5_one_stream_per_rank_world8_kill_rank3():
    out = _run(8, [dict(SMALL, kill=3)])[0]
    for rank, flagged, cks_ok, ok_check, ok_rec, streams in out:
        assert streams == [rank]
        assert flagged == 0 and ok_check
        if rank == 3:
            assert cks_ok is None and ok_rec is None     # the failed rank takes no further part
        else:
            assert cks_ok is True and ok_rec is True     # survivors recover every stream bit-exactly


@pytest.mark.parametrize("i,kill", [(0, 0), (1, 5), (2, None)])
def test_c5_world2_several_streams_per_rank(world2, i, kill):
    for rank, flagged, cks_ok, ok_check, ok_rec, streams in world2[i]:
        assert streams == [m for m in range(8) if m % 2 == rank]
        assert flagged == 0 and ok_check
        if kill is None:
            assert cks_ok is None
        else:
            assert cks_ok is True and ok_rec is True


def test_c5_ragged_positions_world2(world2):
    """Position counts that do not divide evenly among ranks (rows*cols = 15*7),
    and a rank left with no surviving stream after the kill (M = 3, world = 2)."""
    for rank, flagged, cks_ok, ok_check, ok_rec, streams in world2[3]:
        assert flagged == 0 and ok_check and cks_ok is True and ok_rec is True


def test_host_partition_helpers():
    from paper_1604_04740_b200.dist import chunk_bounds, owned_streams

    assert owned_streams(8, 8, 3) == [3]
    assert owned_streams(8, 2, 1) == [1, 3, 5, 7]
    b = chunk_bounds(105, 4)
    assert b[0][0] == 0 and b[-1][1] == 105 and all(b[i][1] == b[i + 1][0] for i in range(3))
