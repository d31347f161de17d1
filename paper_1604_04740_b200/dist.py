"""Multi-GPU orchestration of the hot path (BASELINE configs[4]),
and the partition helpers of C1-C4 (position ranges, the C2 halo exchange,
row ranges, the C4 stream placement and its all_gather).

C5 — "M = 8 streams, one per GPU on 8xB200: entangled GEMM 16384^3 int32 in
[-32, 32), rows sharded; kill one rank's output, recover all streams from the
other 7 via NCCL".  The paper's fault-isolation unit is "a separate processor
core for each of the M streams" (Props 1/3): here stream
m lives on rank m mod world (one stream per GPU when world == M).

Per rank, for each owned stream m (reading R13: stream m = row block m of A):
  1. A_m and A_{m-1} are generated locally from the seed (counter-based, so no
     ring exchange is needed for Eq. 15's c_{m-1}); B is generated locally.
  2. entangle into int8 digit planes (ne_entangle_limbs_stream, a0 + a1),
  3. Delta_m = E_m B on tcgen05 (ne_op_gemm_limbs_stream, a3),
  4. position-major all_to_all: every rank receives all M streams of 1/world of
     the output positions (the only data-path exchange of the check),
  5. disentangle + check on that slice (ne_disentangle_check, a4 + a5),
  6. simulated fail-stop of stream r (its rank's Delta is dropped): the
     survivors exchange again (subgroup all_to_all) and recover every stream
     from the other M-1 (ne_recover, a6),
  7. (verify=True) an order-independent checksum of the checked and the
     recovered outputs, summed over ranks, must agree (bit-exact recovery).

c5_step_failstop is the REAL fail-stop (NEXT-4, world == M): the rank holding
stream plan.kill terminates its process right after its GEMM (os._exit), the
survivors detect it by heartbeat keys in the rendezvous store (a missing key
after `timeout_s` = a dead rank; the first published view wins via
compare_set, so every survivor adopts the same one), shrink the communicator
to the survivors (NCCL: ncclCommShrink with NCCL_SHRINK_ABORT via torch's
shrink_group; gloo: a new world on a fresh store prefix), exchange the M-1
surviving outputs there and recover all M streams (Props 1/3).  With no failure the same step runs the check.
The store must outlive any single rank (torchrun's agent store, or a
TCPStore the launcher hosts); the process that hosts it must not be killed.

The compute backend is injected: ``GpuBackend`` (libne.so kernels) is the
product; the CPU tests drive the same orchestration with a test-only backend
over gloo so the host logic (partitioning, exchange layout, recovery routing)
is exercised without GPUs.  No code here falls back to the CPU by itself.
"""
from __future__ import annotations

import dataclasses
import os
import time
from datetime import timedelta
from typing import Sequence

import torch
import torch.distributed as dist


@dataclasses.dataclass
class C5Plan:
    M: int = 8
    rows_total: int = 16384
    cols: int = 16384
    K: int = 16384
    seed: int = 4
    bound: int = 32          # A, B uniform in [-bound, bound)
    kill: int | None = 3     # stream whose output is lost (None: no fail-stop)

    @property
    def rows(self) -> int:   # rows per stream (row block of A)
        return self.rows_total // self.M


class GpuBackend:
    """The product backend: every call is one libne.so entry point on the
    current CUDA stream."""

    def __init__(self, M: int, bound: int):
        import paper_1604_04740_b200 as ne

        self.ne = ne
        self.cfg = ne.ne_config_for(M)
        self.L, self.limb_bits = ne.ne_gemm_limb_plan(self.cfg, bound)
        self.diag = ne.diag_new()
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.marks = []
        self._bufs = {}
        self.symmetric = None  # exchange windows: symmetric memory if world > 1 (None), or forced on/off

    def _buf(self, key, n, dtype):
        """Step buffers are allocated once and reused (results of a step stay
        valid until the next step that uses the same buffer)."""
        t = self._bufs.get(key)
        if t is None or t.numel() != n or t.dtype != dtype:
            t = torch.empty(n, dtype=dtype, device=self.device)
            self._bufs[key] = t
        return t

    def gen(self, seed, tag, stream, lo, hi, n):
        out = torch.empty(n, dtype=torch.int32, device=self.device)
        self.ne.ne_gen_uniform_i32(seed, tag, stream, lo, hi, out)
        return out

    def prep_b(self, B, K, cols):
        Bt = self._buf("Bt", cols * K, torch.int8)
        self.ne.ne_gemm_prep_b(B, K, cols, Bt, self.diag)
        return Bt

    def entangled_gemm(self, m, A_m, A_prev, Bt, rows, cols, K):
        planes = self._buf("planes", self.L * rows * K, torch.int8)  # stream order: reused per stream
        self.ne.ne_entangle_limbs_stream(self.cfg, m, A_m, A_prev, self.L, planes, self.diag, self.limb_bits)
        out = self._buf(("delta", m), rows * cols, torch.int64)
        self.ne.ne_op_gemm_limbs_stream(self.cfg, planes, self.L, Bt, rows, cols, K, out, self.limb_bits)
        return out

    def exchange_window(self, n: int) -> "SymmWindow":
        """Receive window of n int64 per rank in symmetric memory (collective
        over the world; cached per size)."""
        key = ("win", n)
        w = self._bufs.get(key)
        if w is None:
            w = SymmWindow(n, self.device, self.symmetric)
            self._bufs[key] = w
        return w

    def entangled_gemm_scatter(self, m, A_m, A_prev, Bt, rows, cols, K, dests, keep_local: bool):
        """Entangle + GEMM of stream m with the position-major exchange fused
        into the epilogue: row block j of Delta_m is stored straight into
        dests[j] (receiver j's window, over NVLink); the full Delta_m is also
        kept locally when a recovery exchange may need it."""
        planes = self._buf("planes", self.L * rows * K, torch.int8)
        self.ne.ne_entangle_limbs_stream(self.cfg, m, A_m, A_prev, self.L, planes, self.diag, self.limb_bits)
        out = self._buf(("delta", m), rows * cols, torch.int64) if keep_local else None
        self.ne.ne_op_gemm_limbs_scatter(self.cfg, planes, self.L, Bt, rows, cols, K, list(dests), self.limb_bits,
                                         local=out)
        return out

    def check(self, deltas: Sequence[torch.Tensor], r: int):
        n = deltas[0].numel()
        out = [self._buf(("chk", i), n, torch.int64) for i in range(len(deltas))]
        d = self._buf("diag", 4, torch.int64)
        self.ne.ne_diag_reset(d)
        self.ne.ne_disentangle_check(self.cfg, list(deltas), r, out, None, d)
        return out, int(self.ne.diag_read(d)["fault_positions"])

    def recover(self, deltas: Sequence[torch.Tensor | None], r: int):
        n = next(t for t in deltas if t is not None).numel()
        out = [self._buf(("rec", i), n, torch.int64) for i in range(len(deltas))]
        self.ne.ne_recover(self.cfg, list(deltas), r, out)
        return out

    def sync(self):
        torch.cuda.synchronize()

    def mark(self, name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.marks.append((name, ev))

    def stage_ms(self):
        """Elapsed ms between consecutive marks (after a synchronize)."""
        torch.cuda.synchronize()
        out = {}
        for (_, e0), (name, e1) in zip(self.marks, self.marks[1:]):
            if name not in ("kill", "start"):
                out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
        self.marks = []
        return out


class SymmWindow:
    """A per-rank receive window that every rank can store into: torch
    symmetric memory (peer-mapped over NVLink) when the world has several
    ranks, a plain local buffer for a single rank.  `peer(j)` is rank j's
    window as a tensor on this device; `barrier()` is a device-side barrier on
    the current stream after which every rank's stores into every window are
    visible."""

    def __init__(self, n: int, device, symmetric: bool | None = None):
        world = dist.get_world_size() if dist.is_initialized() else 1
        self.hdl = None
        if not (symmetric if symmetric is not None else world > 1):
            self.local = torch.empty(n, dtype=torch.int64, device=device)
            self.peers = [self.local]
            return
        import torch.distributed._symmetric_memory as symm_mem

        group = dist.group.WORLD
        self.local = symm_mem.empty(n, dtype=torch.int64, device=device)
        self.hdl = symm_mem.rendezvous(self.local, group.group_name)
        self.peers = [self.hdl.get_buffer(j, (n,), torch.int64) for j in range(world)]

    def peer(self, j: int) -> torch.Tensor:
        return self.peers[j]

    def barrier(self):
        if self.hdl is not None:
            self.hdl.barrier(channel=0)


# ---------------------------------------------------------------- C1-C4 partitions
# C1: contiguous position ranges, all M streams of a range on one rank (a1-a5
#     local; the counters are all-reduced after the step).
# C2: contiguous position ranges plus a circular halo of the previous rank's
#     last HALO >= T - 1 entangled positions (one send/recv per stream).
# C3: row ranges of every A_m (all M streams per rank, so the check stays
#     local), B replicated (regenerated from the seed, untimed).
# C4: one entangled stream per rank (world <= M: stream m on rank m mod world;
#     world = k M: stream r // k on rank r, block part r mod k), an all_gather
#     of the per-stream block sums, then each rank checks its block range.
HALO = 64  # >= T - 1 = 63 (C2), even: the rank's own range starts 16-B aligned


def part_range(n: int, parts: int, j: int, align: int = 1) -> tuple[int, int]:
    """[lo, hi) of part j when [0, n) is split into `parts` contiguous ranges
    whose boundaries are multiples of `align` (n itself need not be)."""
    units = -(-n // align)
    lo = min(n, j * units // parts * align)
    hi = min(n, (j + 1) * units // parts * align)
    return lo, hi


def _coll_tensor(t: torch.Tensor, group=None) -> torch.Tensor:
    """gloo collectives take CPU tensors (the NE_BENCH_SHARE_GPU test hook and
    the CPU tests); NCCL takes the CUDA tensor itself."""
    if t.is_cuda and dist.get_backend(group) != "nccl":
        return t.cpu()
    return t


def halo_exchange(ext: Sequence[torch.Tensor], H: int, L: int, group=None) -> None:
    """ext[m] holds positions [lo - H, hi) of stream m (H + L entries, the
    rank's own L from index H).  Fill ext[m][:H] with the previous rank's last
    H positions (circularly: rank 0 receives the last rank's) — one send and
    one receive per stream; with one rank, the stream's own tail."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if L < H:
        raise ValueError(f"halo of {H} positions needs >= {H} positions per rank (got {L})")
    if world == 1:
        for t in ext:
            t[:H].copy_(t[L:L + H])
        return
    rank = dist.get_rank(group)
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    if group is not None:
        nxt, prv = dist.get_global_rank(group, nxt), dist.get_global_rank(group, prv)
    sends = [_coll_tensor(t[L:L + H].contiguous(), group) for t in ext]
    recvs = [torch.empty_like(x) for x in sends]
    ops = []
    for snd, rcv in zip(sends, recvs):
        ops.append(dist.P2POp(dist.isend, snd, nxt, group))
        ops.append(dist.P2POp(dist.irecv, rcv, prv, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    for t, rcv in zip(ext, recvs):
        t[:H].copy_(rcv)


def c4_placement(M: int, world: int, rank: int) -> list[tuple[int, int, int]]:
    """(stream m, block part, parts) items of `rank`: world <= M: every stream
    m with m mod world == rank, whole (1 part); world = k M: stream rank // k,
    part rank mod k of k (each stream on k GPUs, each computing its share of
    the output blocks)."""
    if world <= M:
        return [(m, 0, 1) for m in range(M) if m % world == rank]
    if world % M:
        raise ValueError(f"C4 placement needs world <= M or a multiple of M (M={M}, world={world})")
    k = world // M
    return [(rank // k, rank % k, k)]


def c4_payload(M: int, world: int, rank: int, nb: int) -> list[tuple[int, int, int]]:
    """(m, b_lo, b_hi) block ranges of rank's block sums, in payload order."""
    return [(m, *part_range(nb, k, j)) for m, j, k in c4_placement(M, world, rank)]


def c4_allgather(local: Sequence[torch.Tensor], M: int, nb: int, group=None) -> list[torch.Tensor]:
    """all_gather of every rank's block sums (its c4_payload items, in order):
    returns the M full streams of nb block sums on every rank.  Payloads are
    padded to the largest one; with the placements above every stream ends up
    contiguous in the gathered buffer, so the streams are views of it."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lay = [c4_payload(M, world, r, nb) for r in range(world)]
    width = max(sum(hi - lo for _, lo, hi in it) for it in lay)
    mine = torch.cat(list(local)) if local else torch.empty(0, dtype=torch.int64)
    dev = mine.device
    if mine.numel() < width:
        mine = torch.cat([mine, torch.zeros(width - mine.numel(), dtype=torch.int64, device=dev)])
    if world == 1:
        full = mine
    else:
        snd = _coll_tensor(mine, group)
        full = torch.empty(world * width, dtype=torch.int64, device=snd.device)
        dist.all_gather_into_tensor(full, snd, group=group)
        full = full.to(dev)
    pieces = {m: [] for m in range(M)}
    for r, it in enumerate(lay):
        off = r * width
        for m, lo, hi in it:
            pieces[m].append((lo, off, hi - lo))
            off += hi - lo
    out = []
    for m in range(M):
        ps = sorted(pieces[m])
        lo0, off0, _ = ps[0]
        contiguous = lo0 == 0 and all(ps[i][1] == off0 + ps[i][0] for i in range(len(ps))) and \
            sum(c for _, _, c in ps) == nb
        if contiguous:
            out.append(full[off0:off0 + nb])
        else:
            t = torch.empty(nb, dtype=torch.int64, device=dev)
            for lo, off, c in ps:
                t[lo:lo + c] = full[off:off + c]
            out.append(t)
    return out


# ---------------------------------------------------------------- host logic
def owned_streams(M: int, world: int, rank: int) -> list[int]:
    """Stream m lives on rank m mod world (one stream per GPU when world == M)."""
    return [m for m in range(M) if m % world == rank]


def chunk_bounds(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous near-equal position chunks [lo, hi) of [0, n)."""
    return [(j * n // parts, (j + 1) * n // parts) for j in range(parts)]


def position_major_exchange(local: dict[int, torch.Tensor], M: int, members: list[int], me: int,
                            group=None) -> dict[int, torch.Tensor]:
    """all_to_all so that member j ends with every stream's slice j of the
    positions.  `local` maps stream id -> this rank's full output of that
    stream; every member sends its streams (ascending id) chunk by chunk.
    Returns stream id -> this rank's slice of it."""
    parts = len(members)
    if parts == 1:  # a single rank holds every stream: nothing to move
        return dict(local)
    n = next(iter(local.values())).numel() if local else 0
    n = _bcast_len(n, group)
    bounds = chunk_bounds(n, parts)
    mine = sorted(local)
    send_chunks, send_sizes = [], []
    for (lo, hi) in bounds:
        for m in mine:
            send_chunks.append(local[m][lo:hi])
        send_sizes.append((hi - lo) * len(mine))
    # who owns which streams among the members (static: m mod world over the full world)
    counts = _allgather_counts(len(mine), group)
    ids = _allgather_ids(mine, M, group)
    lo, hi = bounds[members.index(me)]
    recv_sizes = [(hi - lo) * c for c in counts]
    dev = next(iter(local.values())).device if local else _dev(group)
    send = torch.cat(send_chunks) if send_chunks else torch.empty(0, dtype=torch.int64, device=dev)
    send = _coll_tensor(send, group)   # gloo (CPU tests, the share-GPU bench hook): staged through host memory
    recv = torch.empty(sum(recv_sizes), dtype=torch.int64, device=send.device)
    dist.all_to_all_single(recv, send, recv_sizes, send_sizes, group=group)
    recv = recv.to(dev)
    out, off = {}, 0
    for src_ids, c in zip(ids, counts):
        for m in src_ids[:c]:
            out[m] = recv[off:off + (hi - lo)]
            off += hi - lo
    return out


def _bcast_len(n, group):
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return n
    t = torch.tensor([n], dtype=torch.int64, device=_dev(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


def _dev(group):
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _allgather_counts(c, group):
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [c]
    t = torch.tensor([c], dtype=torch.int64, device=_dev(group))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def _allgather_ids(ids, M, group):
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [list(ids)]
    t = torch.full((M,), -1, dtype=torch.int64, device=_dev(group))
    if ids:
        t[: len(ids)] = torch.tensor(ids, dtype=torch.int64)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [[int(v) for v in x.tolist() if v >= 0] for x in out]


def position_checksum(d: Sequence[torch.Tensor], lo: int) -> int:
    """Order-independent checksum of outputs d[m][i] at positions lo + i:
    sum over (m, position) of a 64-bit mix of (value, m, position), wrapping."""
    acc = 0
    for m, t in enumerate(d):
        if t.numel() == 0:
            continue
        pos = torch.arange(lo, lo + t.numel(), dtype=torch.int64, device=t.device)
        z = t * 0x2545F4914F6CDD1D + (pos * 64 + m) * 0x9E3779B97F4A7C15
        z = z ^ (z >> 29)
        acc = (acc + int(z.sum().item())) & (2 ** 64 - 1)
    return acc


def _sum_u64(x: int, group) -> int:
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    # two 32-bit halves so the sum cannot overflow int64 for <= 2^31 ranks
    t = torch.tensor([x & 0xFFFFFFFF, x >> 32], dtype=torch.int64, device=_dev(group))
    dist.all_reduce(t, group=group)
    return (int(t[0].item()) + (int(t[1].item()) << 32)) & (2 ** 64 - 1)


def make_survivor_groups(world: int, M: int):
    """One subgroup per possible dead rank (created collectively up front)."""
    if world < M or world == 1:
        return {}
    return {r: dist.new_group([i for i in range(world) if i != r]) for r in range(world)}


def c5_setup(backend, plan: C5Plan) -> dict:
    """Generate this rank's inputs (outside any timed region): B, and A_m,
    A_{m-1} for every owned stream m, from the counter-based generator."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    M, rows, cols, K, b = plan.M, plan.rows, plan.cols, plan.K, plan.bound
    inp = {"B": backend.gen(plan.seed, 5, 0, -b, b, K * cols), "A": {}}
    for m in owned_streams(M, world, rank):
        inp["A"][m] = (backend.gen(plan.seed, 4, m, -b, b, rows * K),
                       backend.gen(plan.seed, 4, (m - 1) % M, -b, b, rows * K))
    backend.sync()
    return inp


def fused_exchange_ok(plan: C5Plan, world: int) -> bool:
    """The fused GEMM -> exchange needs every rank's position chunk to be a
    whole number of 128-row tiles of each stream's output (and <= 8 ranks)."""
    return world <= 8 and plan.rows % (128 * world) == 0


def c5_step(backend, plan: C5Plan, inp: dict, survivor_groups=None, verify: bool = True,
            exchange: str = "nccl") -> dict:
    """One C5 step on this rank: entangle + GEMM of the owned streams, exchange,
    check, simulated fail-stop of stream plan.kill and recovery (module doc).
    exchange="fused": the GEMM epilogue stores each row block of Delta_m
    straight into its owner's receive window (ne_op_gemm_limbs_scatter over
    symmetric memory) instead of an all_to_all after the GEMM; "nccl": the
    all_to_all.  Stage boundaries are marked with backend.mark(name) (CUDA
    events on GPU)."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    M, rows, cols, K = plan.M, plan.rows, plan.cols, plan.K
    mine = owned_streams(M, world, rank)
    if exchange == "fused" and not fused_exchange_ok(plan, world):
        raise ValueError(f"fused exchange needs rows per stream ({rows}) divisible by 128 x world ({world})")

    backend.mark("start")
    Bt = backend.prep_b(inp["B"], K, cols)
    members = list(range(world))
    if exchange == "fused":
        # GEMM epilogue -> owner's window: rank j receives [M][chunk] (stream-major)
        chunk = rows * cols // world
        win = backend.exchange_window(M * chunk)
        deltas = {}
        for m in mine:
            dests = [win.peer(j)[m * chunk:(m + 1) * chunk] for j in range(world)]
            deltas[m] = backend.entangled_gemm_scatter(m, inp["A"][m][0], inp["A"][m][1], Bt, rows, cols, K, dests,
                                                       keep_local=plan.kill is not None)
        win.barrier()
        backend.mark("entangle_gemm")
        sl = {m: win.local[m * chunk:(m + 1) * chunk] for m in range(M)}
    else:
        deltas = {m: backend.entangled_gemm(m, inp["A"][m][0], inp["A"][m][1], Bt, rows, cols, K) for m in mine}
        backend.mark("entangle_gemm")
        # position-major exchange over all ranks, then the reliability check (r = 0)
        sl = position_major_exchange(deltas, M, members, rank, group=None)
        if world > 1:
            backend.mark("exchange")   # the all_to_all alone (its algbw is reported)
    lo, _ = chunk_bounds(rows * cols, world)[rank]
    d_chk, flagged = backend.check([sl[m] for m in range(M)], 0)
    backend.mark("check" if (exchange != "fused" and world > 1) else "exchange_check")
    total_flags = int(_sum_u64(flagged, None))
    cks_check = _sum_u64(position_checksum(d_chk, lo), None) if verify else None

    result = {"flagged": total_flags, "streams": mine, "check_slice": (lo, d_chk)}
    if plan.kill is None:
        return result

    # simulated fail-stop of stream r: its output never leaves the dead rank
    r = plan.kill
    dead_rank = r % world
    if world == M and world > 1:
        # the whole rank is lost: survivors alone exchange and recover
        if rank == dead_rank:
            result["checksum_ok"] = None  # this rank is the failed one: it takes no further part
            return result
        group = survivor_groups[dead_rank]
        members = [i for i in range(world) if i != dead_rank]
    else:
        group = None
        members = list(range(world))
    backend.mark("kill")
    surviving = {m: v for m, v in deltas.items() if m != r}
    sl2 = position_major_exchange(surviving, M, members, rank, group=group)
    lo2, _ = chunk_bounds(rows * cols, len(members))[members.index(rank)]
    d_rec = backend.recover([None if m == r else sl2[m] for m in range(M)], r)
    backend.mark("exchange_recover")
    if verify:
        cks_rec = _sum_u64(position_checksum(d_rec, lo2), group)
        result["checksum_ok"] = cks_rec == cks_check
    result["recover_slice"] = (lo2, d_rec)
    return result


def c5_run(backend, plan: C5Plan, survivor_groups=None, exchange: str = "nccl") -> dict:
    return c5_step(backend, plan, c5_setup(backend, plan), survivor_groups, exchange=exchange)


# ---------------------------------------------------------------- real fail-stop
def detect_alive(store, epoch: int, world: int, rank: int, timeout_s: float) -> list[int]:
    """Heartbeat round `epoch`: publish this rank's key, wait up to timeout_s
    for the others', then agree on one view (the first one published wins)."""
    store.set(f"ne/alive/{epoch}/{rank}", "1")
    deadline = time.monotonic() + timeout_s
    alive = []
    for r in range(world):
        key = f"ne/alive/{epoch}/{r}"
        while True:
            if store.check([key]):
                alive.append(r)
                break
            if time.monotonic() >= deadline:
                break
            time.sleep(0.01)
    view = ",".join(str(r) for r in alive)
    agreed = store.compare_set(f"ne/view/{epoch}", "", view)
    agreed = agreed.decode() if isinstance(agreed, bytes) else agreed
    return [int(x) for x in agreed.split(",") if x != ""]


def reform_world(store, epoch: int, view: list[int], rank: int, backend_name: str, dead: Sequence[int] = (),
                 api=dist) -> str:
    """Replace the default process group (which includes the dead peer) by one
    over the survivors in `view` (new ranks = positions in `view`).

    NCCL: NCCL's own survivor path — ncclCommShrink of the parent
    communicator with NCCL_SHRINK_ABORT (torch's shrink_group with
    SHRINK_ABORT): the dead rank's outstanding operations are aborted and the
    survivors' communicator is derived from the parent's (no new bootstrap
    through the store); torch makes it the new default group and aborts the
    parent.  Other backends (gloo: the CPU tests) have no shrink: the old
    group is destroyed and a new world is formed on a fresh store prefix.
    Returns "shrink" or "reinit"."""
    if backend_name == "nccl" and hasattr(api, "shrink_group"):
        api.shrink_group(sorted(dead), shrink_flags=api.distributed_c10d.SHRINK_ABORT)
        return "shrink"
    if api.is_initialized():
        api.destroy_process_group()
    prefix = api.PrefixStore(f"ne/world/{epoch}", store)
    api.init_process_group(backend_name, store=prefix, rank=view.index(rank), world_size=len(view),
                           timeout=timedelta(seconds=120))
    return "reinit"


def c5_step_failstop(backend, plan: C5Plan, inp: dict, store, epoch: int = 0, timeout_s: float = 10.0,
                     die: bool = True) -> dict:
    """One C5 step with a real fail-stop (module doc).  world must equal M
    (one stream per rank: a lost rank is a lost stream).  The rank owning
    stream plan.kill exits its process after its GEMM when die is True."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    M, rows, cols, K = plan.M, plan.rows, plan.cols, plan.K
    if world != M:
        raise ValueError("real fail-stop needs one stream per rank (world == M)")
    backend_name = dist.get_backend()
    (m,) = owned_streams(M, world, rank)
    backend.mark("start")
    Bt = backend.prep_b(inp["B"], K, cols)
    delta = backend.entangled_gemm(m, inp["A"][m][0], inp["A"][m][1], Bt, rows, cols, K)
    backend.sync()
    backend.mark("entangle_gemm")
    if die and plan.kill is not None and m == plan.kill:
        os._exit(0)  # fail-stop: the process, its memory and its GPU context are gone
    view = detect_alive(store, epoch, world, rank, timeout_s)
    backend.mark("detect")
    result = {"streams": [m], "view": view}
    if len(view) == world:
        sl = position_major_exchange({m: delta}, M, list(range(world)), rank)
        lo, _ = chunk_bounds(rows * cols, world)[rank]
        d_chk, flagged = backend.check([sl[j] for j in range(M)], 0)
        backend.mark("exchange_check")
        result.update(flagged=int(_sum_u64(flagged, None)), check_slice=(lo, d_chk))
        return result
    dead = [r for r in range(world) if r not in view]
    if len(dead) > 1:
        raise RuntimeError(f"unrecoverable: {len(dead)} streams lost (S:113)")
    r = dead[0]  # stream r == rank r
    how = reform_world(store, epoch, view, rank, backend_name, dead)
    backend.mark("reform")
    members = list(range(len(view)))
    me = view.index(rank)
    sl2 = _exchange_survivors({m: delta}, M, view, me)
    lo2, _ = chunk_bounds(rows * cols, len(view))[me]
    d_rec = backend.recover([None if j == r else sl2[j] for j in range(M)], r)
    backend.mark("exchange_recover")
    result.update(flagged=None, recovered_stream=r, recover_slice=(lo2, d_rec), new_rank=me,
                  new_world=len(members), reform=how)
    return result


def _exchange_survivors(local: dict[int, torch.Tensor], M: int, view: list[int], me: int) -> dict[int, torch.Tensor]:
    """position_major_exchange in the re-formed world (new ranks 0..len(view)-1)."""
    return position_major_exchange(local, M, list(range(len(view))), me, group=None)

