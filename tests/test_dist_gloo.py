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
            plan = C5Plan(**{k: v for k, v in plan_kw.items() if k != "exchange"})
            if plan.M not in groups_for:
                groups_for[plan.M] = make_survivor_groups(world, plan.M)
            exchange = plan_kw.get("exchange", "nccl")
            plan = C5Plan(**{k: v for k, v in plan_kw.items() if k != "exchange"})
            res = c5_run(OracleBackend(plan.M, plan.bound), plan, groups_for[plan.M], exchange=exchange)
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


FUSED = dict(M=8, rows_total=8 * 1024, cols=2, K=3, seed=6, bound=32)


@pytest.mark.parametrize("world,kill", [(8, 3), (2, 5), (4, None)])
def test_c5_fused_exchange(world, kill):
    """exchange="fused": each stream's GEMM stores row block j straight into
    rank j's receive window (the fused GEMM -> exchange kernel's routing;
    gloo emulates the peer stores), then check, simulated fail-stop and
    recovery as in the all_to_all path — every rank's checked and recovered
    slices equal the plain products."""
    out = _run(world, [dict(FUSED, kill=kill, exchange="fused")])[0]
    for rank, flagged, cks_ok, ok_check, ok_rec, streams in out:
        assert flagged == 0 and ok_check
        if kill is None:
            assert cks_ok is None
        elif world == 8 and rank == kill:
            assert cks_ok is None and ok_rec is None
        else:
            assert cks_ok is True and ok_rec is True


def test_fused_exchange_shape_rule():
    from paper_1604_04740_b200.dist import C5Plan, fused_exchange_ok

    assert fused_exchange_ok(C5Plan(), 8)             # C5: 2048 rows per stream = 8 x 256
    assert not fused_exchange_ok(C5Plan(rows_total=8 * 384), 8)
    assert not fused_exchange_ok(C5Plan(), 16)


def test_host_partition_helpers():
    from paper_1604_04740_b200.dist import chunk_bounds, owned_streams

    assert owned_streams(8, 8, 3) == [3]
    assert owned_streams(8, 2, 1) == [1, 3, 5, 7]
    b = chunk_bounds(105, 4)
    assert b[0][0] == 0 and b[-1][1] == 105 and all(b[i][1] == b[i + 1][0] for i in range(3))


# ------------------------------------------------------------------ real fail-stop (NEXT-4)
def _failstop_worker(rank, world, host, port, plan_kw, timeout_s, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from datetime import timedelta

    store = dist.TCPStore(host, port, world, is_master=False, timeout=timedelta(seconds=60))
    dist.init_process_group("gloo", store=dist.PrefixStore("init", store), rank=rank, world_size=world)
    import oracle as O
    from _oracle_backend import OracleBackend
    from paper_1604_04740_b200.dist import C5Plan, c5_setup, c5_step_failstop

    plan = C5Plan(**plan_kw)
    be = OracleBackend(plan.M, plan.bound)
    res = c5_step_failstop(be, plan, c5_setup(be, plan), store, epoch=1, timeout_s=timeout_s)
    M, R, Cc, K, b = plan.M, plan.rows, plan.cols, plan.K, plan.bound
    B = O.gen_uniform(plan.seed, 5, 0, -b, b, K * Cc).reshape(K, Cc)
    plain = np.stack([(O.gen_uniform(plan.seed, 4, m, -b, b, R * K).reshape(R, K) @ B).reshape(-1)
                      for m in range(M)])
    key = "recover_slice" if "recover_slice" in res else "check_slice"
    lo, d = res[key]
    ok = all((d[m].numpy() == plain[m, lo:lo + d[m].numel()]).all() for m in range(M))
    covered = (lo, lo + d[0].numel())
    q.put((rank, key, ok, res["view"], res.get("new_rank"), res.get("flagged"), covered))
    dist.destroy_process_group()


def _run_failstop(world, plan_kw, timeout_s=3.0):
    from datetime import timedelta

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    # the rendezvous store lives in this (launcher) process, so it outlives any rank
    store = dist.TCPStore("127.0.0.1", port, world, is_master=True, timeout=timedelta(seconds=60),
                          wait_for_workers=False)
    procs = [ctx.Process(target=_failstop_worker, args=(r, world, "127.0.0.1", port, plan_kw, timeout_s, q))
             for r in range(world)]
    for p in procs:
        p.start()
    alive = world - (1 if plan_kw.get("kill") is not None else 0)
    out = sorted(q.get(timeout=300) for _ in range(alive))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    del store
    return out


def test_c5_real_failstop_process_exit_world8():
    """The rank holding stream 3 exits its process after its GEMM; the other 7
    detect it by heartbeat timeout, agree on the view, re-form a 7-rank world
    on a fresh store prefix and recover all 8 streams bit-exactly; together
    their slices cover every output position once."""
    out = _run_failstop(8, dict(SMALL, kill=3))
    assert [o[0] for o in out] == [0, 1, 2, 4, 5, 6, 7]
    spans = []
    for rank, key, ok, view, new_rank, flagged, covered in out:
        assert key == "recover_slice" and ok
        assert view == [0, 1, 2, 4, 5, 6, 7] and new_rank == view.index(rank)
        spans.append(covered)
    spans.sort()
    n = SMALL["rows_total"] // SMALL["M"] * SMALL["cols"]
    assert spans[0][0] == 0 and spans[-1][1] == n and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_c5_real_failstop_no_failure_runs_the_check():
    out = _run_failstop(8, dict(SMALL, kill=None))
    for rank, key, ok, view, new_rank, flagged, covered in out:
        assert key == "check_slice" and ok and flagged == 0 and view == list(range(8))


class _FakeDist:
    """Records the calls reform_world makes (no communicator is touched)."""

    class distributed_c10d:
        SHRINK_ABORT, SHRINK_DEFAULT = 1, 0

    def __init__(self, with_shrink=True):
        self.calls = []
        if with_shrink:
            self.shrink_group = lambda ranks, shrink_flags=0: self.calls.append(("shrink_group", ranks, shrink_flags))

    def is_initialized(self):
        self.calls.append(("is_initialized",))
        return True

    def destroy_process_group(self):
        self.calls.append(("destroy_process_group",))

    def PrefixStore(self, prefix, store):  # noqa: N802 (mirrors torch.distributed)
        self.calls.append(("PrefixStore", prefix))
        return (prefix, store)

    def init_process_group(self, backend, store, rank, world_size, timeout):
        self.calls.append(("init_process_group", backend, rank, world_size))


def test_failstop_reform_uses_nccl_shrink_with_abort():
    """f4: on NCCL the survivors take NCCL's own fault path — one
    shrink_group(dead, SHRINK_ABORT) (ncclCommShrink with NCCL_SHRINK_ABORT:
    the parent's pending work aborted, the survivors' communicator derived
    from it) and nothing else; no destroy / re-bootstrap.  Without shrink
    support (gloo) the old world is destroyed and re-formed on a fresh store
    prefix with the survivors' new ranks."""
    from paper_1604_04740_b200.dist import reform_world

    api = _FakeDist()
    view = [0, 1, 2, 4, 5, 6, 7]
    assert reform_world("store", 1, view, 5, "nccl", dead=[3], api=api) == "shrink"
    assert api.calls == [("shrink_group", [3], 1)]
    api = _FakeDist(with_shrink=False)
    assert reform_world("store", 1, view, 5, "nccl", dead=[3], api=api) == "reinit"
    api = _FakeDist()
    assert reform_world("store", 2, view, 5, "gloo", dead=[3], api=api) == "reinit"
    assert api.calls == [("is_initialized",), ("destroy_process_group",), ("PrefixStore", "ne/world/2"),
                         ("init_process_group", "gloo", 4, 7)]


def test_torch_exposes_nccl_shrink():
    """The NCCL survivor path needs torch's shrink_group and the NCCL
    backend's shrink (ncclCommShrink, NCCL >= 2.27; torch bundles 2.28)."""
    assert hasattr(dist, "shrink_group") and hasattr(dist.distributed_c10d, "SHRINK_ABORT")
    assert hasattr(torch._C._distributed_c10d, "ProcessGroupNCCL")
    assert hasattr(torch._C._distributed_c10d.ProcessGroupNCCL, "shrink")
