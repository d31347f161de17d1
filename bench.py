#!/usr/bin/env python
"""bench.py — the entangle -> LSB op -> disentangle + check -> recover hot path
of arXiv 1604.04740 on B200, through libne.so's C ABI.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c2|c2p|c3|c3p|c4|c5]
                    [--impl ours|reference] [--scaling strong|weak] [--configs 0|1]

One "step" is one pass of every §8(a) stage of the chosen BASELINE.json config
over one batch of synthetic (seeded, counter-generated) input that is already
resident in HBM: a0+a1 entangle (range-asserted), a3 the LSB op, a4+a5
disentangle + reliability check, a6 fail-stop recovery of stream (step mod M).
Default workload = configs[2] (C3), the largest single-GPU configuration by
work: the M = 3 entangled 4096^3 integer GEMM on tcgen05 int8 limbs.

Rank 0 prints ONE JSON line (contract in the task statement).  The default
run (C3) also measures C1, C1 at 2^27, C2, C4 and C5 and reports them under
"configs".  Under torchrun (N > 1) every config is partitioned over the ranks
as SURVEY §8(e) specifies (``--scaling strong``, the default: C1 position
ranges, C2 ranges + a halo exchange, C3 row ranges, C4 one stream per GPU +
an all_gather, C5 one stream per rank) or replicated (``--scaling weak``);
timing is the max over ranks of CUDA-event time, value = the whole job's work
per step / that time.  Every line compares its timed outputs with the oracle
at sampled positions (correctness.oracle_rows_equal).  ``--impl reference``
times the CPU oracle (oracle/, plain C, 1 core) on a bounded sample of the
same workload; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK), "fallback (B200_PROFILING.md)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    return json.load(open(p)) if os.path.exists(p) else {}


# ====================================================================== workloads
class Workload:
    """A BASELINE.json config: buffers, one step as a list of named stages."""

    name = ""
    metric_unit = ""
    launches_per_step = 0

    def stages(self, i):  # -> list of (stage_name, callable)
        raise NotImplementedError

    # independent stages run side by side inside the timed step: {side stage: the stage it runs beside}
    # (the side stage on a second stream, forked before and joined after the main one; the stage
    # timings keep every stage on its own)
    concurrent: dict = {}
    overlap = True

    def run_step(self, i):
        st = self.stages(i)
        fns = dict(st)
        par = self.concurrent if self.overlap else {}
        beside = {}
        for side, mains in par.items():
            main = next((m for m in (mains if isinstance(mains, tuple) else (mains,)) if m in fns), None)
            if side in fns and main is not None:
                beside[main] = side
        sides = set(beside.values())
        torch = self.torch
        for nm, f in st:
            if nm in sides:
                continue
            if nm not in beside:
                f()
                continue
            cur = torch.cuda.current_stream()
            if getattr(self, "_side", None) is None:
                self._side = torch.cuda.Stream()
            fork, join = torch.cuda.Event(), torch.cuda.Event()
            fork.record(cur)
            self._side.wait_event(fork)
            with torch.cuda.stream(self._side):
                fns[beside[nm]]()
            f()
            join.record(self._side)
            cur.wait_event(join)

    # ---- end to end (pinned host inputs -> device -> result -> pinned host),
    # pipelined across steps: step i's H2D, compute and D2H run on three CUDA
    # streams over two device buffer slots, so the copies of one step overlap
    # the compute of another and H2D overlaps D2H (PCIe is full duplex).
    # Every step still moves all of its inputs and results.
    E2E_IN: tuple = ()
    E2E_OUT: tuple = ()
    def e2e_bytes(self):
        def flat(v):
            return list(v) if isinstance(v, (list, tuple)) else [v]
        return sum(t.numel() * t.element_size() for n in self.E2E_IN + self.E2E_OUT for t in flat(getattr(self, n)))

    @property
    def E2E_PIPELINE(self):  # pipelining pays once the copies outweigh its per-step enqueue cost
        return self.e2e_bytes() > (8 << 20)

    def e2e(self, steps):
        return self.e2e_pipeline(steps) if self.E2E_PIPELINE else self.e2e_serial(steps)

    def e2e_serial(self, steps):
        """One stream: H2D inputs, the step, D2H results, in order."""
        torch = self.torch

        def flat(v):
            return list(v) if isinstance(v, (list, tuple)) else [v]

        dev_in = [t for n in self.E2E_IN for t in flat(getattr(self, n))]
        dev_out = [t for n in self.E2E_OUT for t in flat(getattr(self, n))]
        h_in = [t.cpu().pin_memory() for t in dev_in]
        h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in dev_out]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        for i in range(steps):
            for d, h in zip(dev_in, h_in):
                d.copy_(h, non_blocking=True)
            self.run_step(i)
            for h, d in zip(h_out, dev_out):
                h.copy_(d, non_blocking=True)
        t1.record()
        torch.cuda.synchronize()
        return (t0.elapsed_time(t1) / steps, sum(h.numel() * h.element_size() for h in h_in),
                sum(h.numel() * h.element_size() for h in h_out))

    def e2e_pipeline(self, steps, nslots=2):
        torch = self.torch

        def flat(v):
            return list(v) if isinstance(v, (list, tuple)) else [v]

        names = self.E2E_IN + self.E2E_OUT
        orig = {n: getattr(self, n) for n in names}
        slots = [orig] + [{n: ([t.clone() for t in orig[n]] if isinstance(orig[n], list) else orig[n].clone())
                           for n in names} for _ in range(nslots - 1)]
        h_in = {n: [t.cpu().pin_memory() for t in flat(orig[n])] for n in self.E2E_IN}
        h_out = [{n: [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in flat(orig[n])]
                  for n in self.E2E_OUT} for _ in range(nslots)]
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        ev_in, ev_cmp, ev_out = [mk() for _ in range(steps)], [mk() for _ in range(steps)], [mk() for _ in range(steps)]
        t0, t1 = mk(), mk()
        torch.cuda.synchronize()
        t0.record(s_in)
        for i in range(steps):
            k = i % nslots
            sl = slots[k]
            with torch.cuda.stream(s_in):
                if i >= nslots:
                    s_in.wait_event(ev_cmp[i - nslots])  # compute i-nslots done reading slot k's inputs
                for n in self.E2E_IN:
                    for d, h in zip(flat(sl[n]), h_in[n]):
                        d.copy_(h, non_blocking=True)
                ev_in[i].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[i])
                if i >= nslots:
                    s_cmp.wait_event(ev_out[i - nslots])  # D2H i-nslots done reading slot k's results
                for n in names:
                    setattr(self, n, sl[n])
                self.run_step(i)
                ev_cmp[i].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[i])
                for n in self.E2E_OUT:
                    for h, d in zip(h_out[k][n], flat(sl[n])):
                        h.copy_(d, non_blocking=True)
                ev_out[i].record(s_out)
        t1.record(s_out)
        torch.cuda.synchronize()
        for n in names:
            setattr(self, n, orig[n])
        h2d = sum(h.numel() * h.element_size() for n in self.E2E_IN for h in h_in[n])
        d2h = sum(h.numel() * h.element_size() for n in self.E2E_OUT for h in h_out[0][n])
        return t0.elapsed_time(t1) / steps, h2d, d2h

    def _time(self, fn, reps):
        """ms per call of fn, captured once in a CUDA graph and replayed: the
        same launch path as the timed step, so plain and entangled compare
        (eager launches when the step holds a collective, as the timed run)."""
        torch = self.torch
        fn()
        torch.cuda.synchronize()
        if getattr(self, "eager_only", False):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def work_per_step(self):  # metric units per step of THIS rank (before /time)
        raise NotImplementedError

    # ---- multi-GPU: "strong" partitions the stated problem
    # over the ranks (value = the whole problem / max-over-ranks time);
    # "weak" runs one independent replica per rank (per-rank seeds)
    partitioned = False
    has_collective = False   # a collective inside the step (timed eagerly: not graph-captured)
    partition_note = "single GPU: the whole problem on one rank"

    def setup_partition(self, rank, world, scaling, seed):
        self.rank, self.world = rank, world
        self.partitioned = scaling == "strong" and world > 1
        return seed + 1000 * rank if (scaling == "weak" and world > 1) else seed

    def job_work(self):
        """Metric units of the whole job per step (all ranks)."""
        if self.partitioned:
            return self.global_work()
        return self.work_per_step() * getattr(self, "world", 1)

    def stage_info(self):  # stage -> (bound, algorithmic amount per launch, unit)
        raise NotImplementedError


class C3Gemm(Workload):
    # B's digit planes do not depend on A's entangle (or ABFT's encode), nor the fail-stop recovery on the check
    concurrent = {"prep_b": ("entangle", "encode"), "recover": "check"}
    """configs[2]: M=3 entangled GEMM, A_m 4096x4096 int32 in [-64,64), shared B
    4096x4096 in [-64,64), K = 4096, int64 results; tcgen05 int8 limbs (L = 4)."""

    name = "C3"
    metric_unit = "Gop/s"
    E2E_IN = ("A", "B")
    E2E_OUT = ("dout",)

    def __init__(self, rank, n=4096, seed=2, algo="tc", scheme="entangled", limbs="plan", fuse=True,
                 paper_shape=None, world=1, scaling="strong", abound=64, bbound=64):
        import torch
        import paper_1604_04740_b200 as ne
        from paper_1604_04740_b200.dist import part_range

        self.ne, self.torch = ne, torch
        self.M, self.rows, self.cols, self.K = 3, n, n, n
        self.true_shape = None
        if paper_shape is not None:
            # the paper's GEMM experiment: M subblocks of 2000 x N times N x 1200;
            # operands zero-padded to the kernel's tile multiples (rows 128, cols 256, K 128),
            # the metric counts the true shape only
            Mp, Rt, Ct, Kt = paper_shape
            self.M, self.true_shape = Mp, (Rt, Ct, Kt)
            self.rows, self.cols, self.K = -(-Rt // 128) * 128, -(-Ct // 256) * 256, -(-Kt // 128) * 128
            self.name = f"C3P_M{Mp}_N{Kt}"
        if scaling == "strong" and world > 1 and (paper_shape is not None or self.rows % (256 * world)):
            scaling = "weak"
            self.partition_note = "replicas (the row split needs whole 256-row pair bands per rank)"
        self.seed = self.setup_partition(rank, world, scaling, seed)
        self.rows_global, self.r0 = self.rows, 0
        if self.partitioned:
            # rows of every A_m split over the ranks (all M streams per rank: the check stays local);
            # B replicated, generated from the seed on every rank outside the timing
            self.r0, r1 = part_range(self.rows, world, rank, 256)
            self.rows = r1 - self.r0
            self.partition_note = (f"rows [{self.r0}, {r1}) of every A_m (all M = {self.M} streams) on rank {rank} "
                                   f"of {world}; B replicated (regenerated from the seed, untimed); no collective in "
                                   "the step, counters all-reduced after it")
        self.cfg = ne.ne_config_for(self.M)
        # operand ranges: C3's U[-64, 64) by default; wider ranges (--abound / --bbound) take the
        # general digit plan of ne_gemm_plan_for (split or base-256 planes of A, B in base-256 planes)
        self.abound, self.bbound = abound, bbound
        self.wide = (abound, bbound) != (64, 64) and algo == "tc" and scheme == "entangled"
        self.LB = 1
        if self.wide:
            self.plan = ne.ne_gemm_plan_for(self.cfg, abound, bbound)
            self.L, self.limb_bits, self.LB = self.plan.LA, self.plan.digit_bits, self.plan.LB
            self.name = f"C3_a{abound}_b{bbound}"
            fuse = False
        elif limbs == "base256":
            self.L, self.limb_bits = ne.ne_gemm_limbs_for(self.cfg, 64), 8
        else:  # the cheapest exact plan: base 2^l, 2 limbs (|A| < 128)
            self.L, self.limb_bits = ne.ne_gemm_limb_plan(self.cfg, 64)
        self.algo = algo
        if algo != "tc":
            self.name = f"{self.name}_{algo}"   # traffic.json key of the CUDA-core lines
        self.scheme = scheme
        # disentangle + check fused into the GEMM epilogue (ne_op_gemm_limbs_check)
        self.fuse = bool(fuse) and algo == "tc" and scheme == "entangled"
        M, R, Cc, K, L = self.M, self.rows, self.cols, self.K, self.L
        dev = "cuda"
        if self.true_shape is None:
            self.A = [torch.empty(R * K, dtype=torch.int32, device=dev) for _ in range(M)]
            for m in range(M):
                ne.ne_gen_uniform_i32(self.seed, 4, m, -abound, abound, self.A[m], self.r0 * K)
            self.B = torch.empty(K * Cc, dtype=torch.int32, device=dev)
            ne.ne_gen_uniform_i32(self.seed, 5, 0, -bbound, bbound, self.B)
        else:
            Rt, Ct, Kt = self.true_shape
            self.A = [torch.zeros(R * K, dtype=torch.int32, device=dev) for _ in range(M)]
            for m in range(M):
                t = torch.empty(Rt * Kt, dtype=torch.int32, device=dev)
                ne.ne_gen_uniform_i32(self.seed, 4, m, -64, 64, t)
                self.A[m].view(R, K)[:Rt, :Kt] = t.view(Rt, Kt)
            self.B = torch.zeros(K * Cc, dtype=torch.int32, device=dev)
            t = torch.empty(Kt * Ct, dtype=torch.int32, device=dev)
            ne.ne_gen_uniform_i32(self.seed, 5, 0, -64, 64, t)
            self.B.view(K, Cc)[:Kt, :Ct] = t.view(Kt, Ct)
        self.planes = torch.empty(M * L * R * K, dtype=torch.int8, device=dev)
        self.Bt = torch.empty(self.LB * Cc * K, dtype=torch.int8, device=dev)
        self.delta = [torch.empty(R * Cc, dtype=torch.int64, device=dev) for _ in range(M)]
        self.dout = [torch.empty(R * Cc, dtype=torch.int64, device=dev) for _ in range(M)]
        self.drec = [torch.empty(R * Cc, dtype=torch.int64, device=dev) for _ in range(M)]
        self.bitmap = torch.empty(R * Cc // 32, dtype=torch.int32, device=dev)
        self.diag = ne.diag_new()
        if algo in ("imad", "imad64"):
            self.eps = [torch.empty(R * K, dtype=torch.int64, device=dev) for _ in range(M)]
        self.launches_per_step = 4 if self.fuse else 5
        if self.wide:   # the plan's GEMM is one launch per (group of <= 4 A planes, B plane)
            self.launches_per_step = 4 + -(-self.L // 4) * self.LB
        if algo in ("imad", "imad64"):   # entangle, GEMM, check, recover
            self.launches_per_step = 4
        self.counters = torch.zeros(ne.ne_gemm_check_workspace(R, Cc) // 4, dtype=torch.int32, device=dev)
        if scheme == "abft":
            # the paper's comparison method on the same kernels: plain data (1 int8
            # limb), one checksum stream (Eq. 4; |sum| <= 192 -> 2 limbs)
            self.Asum = torch.empty(R * K, dtype=torch.int32, device=dev)
            self.pdata = torch.empty(M * R * K, dtype=torch.int8, device=dev)
            self.psum = torch.empty(2 * R * K, dtype=torch.int8, device=dev)
            self.e = torch.empty(R * Cc, dtype=torch.int64, device=dev)
            self.launches_per_step = 6
            del self.planes

    def stages(self, i):
        ne, cfg, M = self.ne, self.cfg, self.M
        r = i % M
        part = [None if m == r else self.delta[m] for m in range(M)]
        if self.scheme == "abft":
            rr = [None if m == r else self.delta[m] for m in range(M)]
            return [
                ("encode", lambda: ne.ne_abft_encode_limbs(cfg, self.A, self.pdata, 2, self.psum, self.diag)),
                ("prep_b", lambda: ne.ne_gemm_prep_b(self.B, self.K, self.cols, self.Bt, self.diag)),
                ("gemm", lambda: (ne.ne_op_gemm_limbs(cfg, self.pdata, 1, self.Bt, self.rows, self.cols, self.K,
                                                      self.delta),
                                  ne.ne_op_gemm_limbs_stream(cfg, self.psum, 2, self.Bt, self.rows, self.cols,
                                                             self.K, self.e))),
                ("check", lambda: ne.ne_abft_check(cfg, self.delta, self.e, self.bitmap, self.diag)),
                ("recover", lambda: ne.ne_abft_recover(cfg, rr, self.e, r, self.drec[r])),
            ]
        if self.algo in ("imad", "imad64"):
            # CUDA-core comparison point: one IMAD.WIDE (32 x 32 -> 64) per MAC — C3's entangled
            # operand fits int32 (|eps| <= 64 (2^22 + 1)) — or the any-operand 64-bit form
            ia = ne.NE_GEMM_IMAD32W if self.algo == "imad" else ne.NE_GEMM_IMAD64
            return [
                ("entangle", lambda: ne.ne_entangle(cfg, self.A, self.eps, self.diag)),
                ("gemm", lambda: ne.ne_op_gemm(cfg, self.eps, self.B, self.rows, self.cols, self.K, self.delta,
                                               algo=ia, diag=self.diag)),
                ("check", lambda: ne.ne_disentangle_check(cfg, self.delta, 0, self.dout, self.bitmap, self.diag)),
                ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec)),
            ]
        if self.wide:
            return [
                ("entangle", lambda: ne.ne_entangle_plan(cfg, self.A, self.plan, self.planes, self.diag)),
                ("prep_b", lambda: ne.ne_gemm_prep_b_planes(self.B, self.K, self.cols, self.LB, self.Bt, self.diag)),
                ("gemm", lambda: ne.ne_op_gemm_plan(cfg, self.planes, self.plan, self.Bt, self.rows, self.cols, self.K,
                                                    self.delta)),
                ("check", lambda: ne.ne_disentangle_check(cfg, self.delta, 0, self.dout, self.bitmap, self.diag)),
                ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec)),
            ]
        if self.fuse:
            return [
                ("entangle", lambda: ne.ne_entangle_limbs(cfg, self.A, self.L, self.planes, self.diag,
                                                          self.limb_bits)),
                ("prep_b", lambda: ne.ne_gemm_prep_b(self.B, self.K, self.cols, self.Bt, self.diag)),
                ("gemm_check", lambda: ne.ne_op_gemm_limbs_check(cfg, self.planes, self.L, self.Bt, self.rows,
                                                                 self.cols, self.K, self.delta, 0, self.dout,
                                                                 self.counters, self.bitmap, self.diag,
                                                                 self.limb_bits)),
                ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec)),
            ]
        return [
            ("entangle", lambda: ne.ne_entangle_limbs(cfg, self.A, self.L, self.planes, self.diag, self.limb_bits)),
            ("prep_b", lambda: ne.ne_gemm_prep_b(self.B, self.K, self.cols, self.Bt, self.diag)),
            ("gemm", lambda: ne.ne_op_gemm_limbs(cfg, self.planes, self.L, self.Bt, self.rows, self.cols, self.K,
                                                 self.delta, self.limb_bits)),
            ("check", lambda: ne.ne_disentangle_check(cfg, self.delta, 0, self.dout, self.bitmap, self.diag)),
            ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec)),
        ]

    def work_per_step(self):
        R, Cc, K = self.true_shape or (self.rows, self.cols, self.K)
        return 2 * self.M * R * Cc * K / 1e9  # G int64-equivalent ops (true shape)

    def global_work(self):
        return 2 * self.M * self.rows_global * self.cols * self.K / 1e9

    def stage_info(self):
        M, R, Cc, K, L = self.M, self.rows, self.cols, self.K, self.L
        n = R * Cc
        if self.scheme == "abft":
            return {"encode": ("hbm", R * K * (M * 4 + M + 2) / 1e9, "GB"),
                    "prep_b": ("hbm", K * Cc * 5 / 1e9, "GB"),
                    "gemm": ("tensor", 2 * (M + 2) * R * Cc * K / 1e12, "TOP"),
                    "check": ("hbm", (M + 1) * n * 8 / 1e9, "GB"),
                    "recover": ("hbm", (M + 1) * n * 8 / 1e9, "GB")}
        Rt, Ct, Kt = self.true_shape or (R, Cc, K)  # useful work only (the zero padding is not counted)
        gemm = ("tensor", 2 * L * self.LB * M * Rt * Ct * Kt / 1e12, "TOP") if self.algo == "tc" else \
            ("alu", M * Rt * Ct * Kt / 1e12, "TMAC")
        return {
            "entangle": ("hbm", M * R * K * (4 + (L if self.algo == "tc" else 8)) / 1e9, "GB"),
            "prep_b": ("hbm", K * Cc * (4 + self.LB) / 1e9, "GB"),
            "gemm": gemm,
            "gemm_check": gemm,  # fused: the tensor work bounds it; + M*n*8 B of d_hat written under it
            "check": ("hbm", (M * n * 16 + n / 8) / 1e9, "GB"),
            "recover": ("hbm", ((M - 1) * n * 8 + M * n * 8) / 1e9, "GB"),
        }

    def config(self):
        wl = ("C3 (BASELINE configs[2]): M=3 entangled GEMM A_m 4096x4096 int32 U[-64,64), "
              "shared B 4096x4096 U[-64,64), K=4096, int64 results")
        if self.wide:
            p = self.plan
            wl = (f"C3 shape with wider operands: M=3 entangled GEMM A_m 4096x4096 int32 U[-{self.abound},"
                  f"{self.abound}), shared B U[-{self.bbound},{self.bbound}), K=4096, int64 results; digit plan "
                  f"{'split' if p.kind else 'eps'} LA={p.LA} (bit weights {list(p.a_shift)[:p.LA]}) x LB={p.LB}")
        if self.true_shape is not None:
            Rt, Ct, Kt = self.true_shape
            wl = (f"C3P (the paper's GEMM shape, P:1119-1121): M={self.M} subblocks of {Rt}x{Kt} int32 "
                  f"U[-64,64) times a shared {Kt}x{Ct}, int64 results; zero-padded to {self.rows}x{self.K} "
                  f"x {self.K}x{self.cols} for the tiles, metric on the true shape")
        return {"workload": wl,
                "M": self.M, "rows": self.rows, "cols": self.cols, "K": self.K,
                "limbs_L": self.L if self.algo == "tc" else None, "gemm_algo": self.algo,
                "limb_base_bits": self.limb_bits if self.algo == "tc" else None,
                "scheme": self.scheme + (" (ABFT single checksum stream, Eqs. 3-6: the paper's comparison method)"
                                         if self.scheme == "abft" else " (numerical entanglement)"),
                "entanglement": {"l": self.cfg.l, "k": self.cfg.k, "w": 64},
                "l2": "working set ~1.9 GB per step >> 126 MB L2 (no flush needed)",
                "step": ("entangle(limbs)+prep_B+GEMM with fused disentangle/check(r=0)+recover(r=step mod 3)"
                         if self.fuse else
                         "entangle(limbs)+prep_B+GEMM+disentangle/check(r=0)+recover(r=step mod 3)")}

    def plain_times(self, reps=10):
        """The paper's comparison (F5) with matched scopes, each
        pipeline captured as one CUDA graph and replayed like the timed step:
          no-fault entangled: entangle(limbs) + prep_B + GEMM + disentangle/check
          plain, same kernel: int32 -> int8 planes (L digit planes, the upper
            ones 0) + prep_B + the same tcgen05 GEMM kernel and plan
          plain, native:      int32 -> one int8 plane + prep_B + the 1-digit
            tcgen05 GEMM (the narrowest exact plain form)
        and the fail-stop cost (recovery alone) separately; both sides strictly in
        order (no side stream, unlike the timed step).  Also cuBLASLt's
        int8 x int8 -> int32 GEMM on the same multiply-adds (torch._int_mm) as
        a library context number (int32 output, no int64 recombination)."""
        torch, ne = self.torch, self.ne
        if self.algo != "tc" or self.scheme != "entangled" or self.wide:
            return {}
        M, R, Cc, K, L = self.M, self.rows, self.cols, self.K, self.L
        cfg = self.cfg
        out = {}
        stl = self.stages(0)
        st = dict(stl)
        out["entangled_nofault"] = (self._time(lambda: [f() for nm, f in stl if nm != "recover"], reps),
                                    "+".join(nm for nm, _ in stl if nm != "recover"))
        out["failstop_recover"] = (self._time(st["recover"], reps), "recover(one stream lost)")
        scratch = [torch.empty(R * Cc, dtype=torch.int64, device="cuda") for _ in range(M)]
        for tag, Lp, b in (("plain_same_kernel", L, self.limb_bits), ("plain_L1_int64_out", 1, 8)):
            planes = torch.empty(M * Lp * R * K, dtype=torch.int8, device="cuda")
            kern = ne.ne_gemm_kernel_for(cfg, Lp, b, R, Cc, K)

            def run(planes=planes, Lp=Lp, b=b):
                ne.ne_to_limbs(self.A, Lp, planes, self.diag)
                ne.ne_gemm_prep_b(self.B, K, Cc, self.Bt, self.diag)
                ne.ne_op_gemm_limbs(cfg, planes, Lp, self.Bt, R, Cc, K, scratch, b)
            out[tag] = (self._time(run, reps), f"int32->int8 planes (L={Lp})+prep_B+GEMM(L={Lp}, {kern} kernel, "
                                               f"int64 out)")
            out[tag + "_gemm_only"] = (self._time(
                lambda planes=planes, Lp=Lp, b=b: ne.ne_op_gemm_limbs(cfg, planes, Lp, self.Bt, R, Cc, K, scratch, b),
                reps), f"GEMM(L={Lp}) alone")
            del planes
        # the narrowest native form: one int8 digit, int32 products (what a plain int8 GEMM returns)
        if R % 256 == 0 and Cc % 256 == 0:
            p1 = torch.empty(M * R * K, dtype=torch.int8, device="cuda")
            o32 = [torch.empty(R * Cc, dtype=torch.int32, device="cuda") for _ in range(M)]

            def run1():
                ne.ne_to_limbs(self.A, 1, p1, self.diag)
                ne.ne_gemm_prep_b(self.B, K, Cc, self.Bt, self.diag)
                ne.ne_op_gemm_plain_i32(p1, self.Bt, R, Cc, K, o32)
            out["plain_native_L1"] = (self._time(run1, reps), "int32->int8 plane (L=1)+prep_B+GEMM(L=1, pair kernel, "
                                                               "int32 out)")
            out["plain_native_L1_gemm_only"] = (self._time(lambda: ne.ne_op_gemm_plain_i32(p1, self.Bt, R, Cc, K, o32),
                                                           reps), "GEMM(L=1, int32 out) alone")
            del p1, o32
        del scratch
        try:  # library context: cuBLASLt int8 GEMM, int32 out, the same M x rows x cols x K multiply-adds
            a8 = torch.randint(-64, 64, (M * R, K), dtype=torch.int8, device="cuda")
            b8 = torch.randint(-64, 64, (K, Cc), dtype=torch.int8, device="cuda")
            out["context_cublaslt_int8"] = (self._time(lambda: torch._int_mm(a8, b8), reps),
                                            "torch._int_mm (cuBLASLt) int8 x int8 -> int32, one (M*rows) x K x cols GEMM")
            del a8, b8
        except Exception as e:  # noqa: BLE001 — context only
            out["context_cublaslt_int8"] = (None, f"unavailable: {type(e).__name__}")
        return out

    # ---- CPU oracle on a bounded sample (rows of every stream)
    def sample_rows(self, rows_sample):
        """One row per 256-row pair band (C3: 16 bands), its 32-row TMEM lane
        group cycling through all 8 (both CTA halves, every epilogue quarter);
        the paper shapes: the first rows of the true (unpadded) operand."""
        if self.true_shape is not None:
            return np.arange(rows_sample)
        band = max(32, self.rows // rows_sample)
        return np.array([(band * i + 32 * (i % 8) % band + (7 * i) % 32) % self.rows for i in range(rows_sample)])

    def oracle_sample(self, rows_sample):
        import oracle as O

        M, K, Cc = self.M, self.K, self.cols
        if self.true_shape is not None:
            _, Cc, K = self.true_shape
        rows = self.sample_rows(rows_sample)
        ocfg = O.config_for(M, 64)
        ab, bb = getattr(self, "abound", 64), getattr(self, "bbound", 64)
        A = np.stack([np.concatenate([O.gen_uniform(self.seed, 4, m, -ab, ab, K, (self.r0 + int(r)) * K)
                                      for r in rows]) for m in range(M)])
        B = O.gen_uniform(self.seed, 5, 0, -bb, bb, K * Cc).reshape(K, Cc)
        t0 = time.perf_counter()
        E = O.entangle(ocfg, A)
        D = O.op_gemm(ocfg, E.reshape(M, len(rows), K), B).reshape(M, -1)
        d, flags, nf = O.disentangle_check(ocfg, D, 0)
        O.recover(ocfg, [None] + [D[m] for m in range(1, M)], 0)
        dt = time.perf_counter() - t0
        self._oref = (rows, D.reshape(M, len(rows), Cc), d.reshape(M, len(rows), Cc))
        return dt, 2 * M * len(rows) * Cc * K / 1e9, \
            f"{len(rows)} of {self.rows} rows of each of the M={M} streams (one per 256-row band, all 8 TMEM " \
            f"lane groups), full K and cols (same seeded inputs)"

    def oracle_compare(self):
        """The oracle's delta and d_hat of the sampled rows vs the timed run's."""
        if getattr(self, "_oref", None) is None or self.scheme != "entangled":
            return None
        rows, D, d = self._oref
        idx = self.torch.from_numpy(rows).cuda()
        ct = D.shape[-1]
        got_d = np.stack([t.view(self.rows, self.cols)[idx, :ct].cpu().numpy() for t in self.delta])
        got = np.stack([t.view(self.rows, self.cols)[idx, :ct].cpu().numpy() for t in self.dout])
        return bool((got_d == D).all() and (got == d).all())


class C4PermInner(Workload):
    """configs[3]: M=4 streams of 2^28 int32 U[-2^12, 2^12): permutation by a
    seeded bijection, then inner products with a shared 1024-vector in blocks
    of 1024; HBM-bound.  eps at rest in the AoS layout (one 32-B sector per
    position), gather + inner + disentangle/check fused."""

    name = "C4"
    metric_unit = "GB/s"
    E2E_IN = ("c",)
    E2E_OUT = ("dout",)

    def __init__(self, rank, n=1 << 28, seed=3, layout="aos", w=64, world=1, scaling="strong", algo="bucket"):
        import torch
        import paper_1604_04740_b200 as ne

        self.ne, self.torch = ne, torch
        self.M, self.n, self.B, self.layout, self.w = 4, n, 1024, layout, w
        self.algo = algo if (layout == "aos" and w == 64) else "gather"
        self.b0 = 0   # first output block this rank checks
        if scaling == "strong" and world > 1 and (layout != "aos" or w != 64):
            scaling = "weak"
            self.partition_note = "replicas (the stream placement is built for the default w = 64 layout)"
        if scaling == "strong" and world > 1:
            self.algo = "gather"   # the placement gathers per stream (ne_op_permute_inner_stream)
            self._init_placement(rank, world, seed)
            return
        if layout != "aos":
            self.name = "C4_soa"
        # w = 32 containers (NEXT-3): C4's own range (block sums up to 2^34) does
        # not fit 32 bits, so the w = 32 line uses 7-bit inputs and coefficients
        # (|block sum| <= 1024 * 64 * 64 = 2^22 < 8 323 072, the M = 4, w = 32 range)
        self.vr = (1 << 12) if w == 64 else 64
        if w == 32:
            self.name = "C4_w32"
        self.seed = seed + 1000 * rank
        self.cfg = ne.ne_config_for(4, w)
        dev = "cuda"
        self.c = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(4)]
        for m in range(4):
            ne.ne_gen_uniform_i32(self.seed, 1, m, -self.vr, self.vr, self.c[m])
        self.perm = torch.empty(n, dtype=torch.int32, device=dev)
        ne.ne_gen_perm_i32(self.seed, 6, self.perm)
        self.v = torch.empty(self.B, dtype=torch.int32, device=dev)
        ne.ne_gen_uniform_i32(self.seed, 7, 0, -self.vr, self.vr, self.v)
        wd = torch.int64 if w == 64 else torch.int32
        if layout == "aos":
            self.eps = torch.empty(n * 4, dtype=wd, device=dev)
        else:  # SoA: one int64 stream per m (each gathered position touches 4 sectors)
            self.eps = [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(4)]
        self.nb = n // self.B
        self.delta = [torch.empty(self.nb, dtype=wd, device=dev) for _ in range(4)]
        self.dout = [torch.empty(self.nb, dtype=wd, device=dev) for _ in range(4)]
        self.drec = [torch.empty(self.nb, dtype=wd, device=dev) for _ in range(4)]
        self.bitmap = torch.empty((self.nb + 31) // 32, dtype=torch.int32, device=dev)
        self.diag = ne.diag_new()
        self.launches_per_step = 3
        if self.algo == "gather" and layout == "aos" and w == 64:
            self.name = "C4_gather"   # traffic.json key of the gather-kernel line
        if self.algo == "bucket":
            self.ws = torch.empty(ne.ne_permute_inner_workspace(self.cfg, n, self.B), dtype=torch.uint8, device=dev)
            self.launches_per_step = 5   # entangle, scatter, reduce, check, recover (+ memsets)

    def _init_placement(self, rank, world, seed):
        """one entangled stream per GPU (streams m = rank mod
        world when world <= M; at world = 2M each stream on 2 GPUs, each
        computing half of its output blocks).  The global permutation stays
        local to a stream (every rank holds pi and its streams' eps in full:
        no all-to-all over 2^28 elements); c_{m-1} for Eq. 15 is regenerated
        from the seed.  After the gathers, an all_gather of the per-stream
        block sums (M x 2^18 int64) gives every rank all M streams of every
        block, and rank r checks and recovers its own range of blocks."""
        import torch
        from paper_1604_04740_b200.dist import c4_payload, part_range

        ne, n, M = self.ne, self.n, self.M
        self.seed = self.setup_partition(rank, world, "strong", seed)
        self.cfg = ne.ne_config_for(M, 64)
        self.vr = 1 << 12
        self.nb = n // self.B
        self.items = c4_payload(M, world, rank, self.nb)
        self.owned = sorted({m for m, _, _ in self.items})
        need = sorted(set(self.owned) | {(m - 1) % M for m in self.owned})
        dev = "cuda"
        self.cgen = {}
        for m in need:
            t = torch.empty(n, dtype=torch.int32, device=dev)
            ne.ne_gen_uniform_i32(self.seed, 1, m, -self.vr, self.vr, t)
            self.cgen[m] = t
        self.c = [self.cgen[m] for m in need]   # the step's inputs (e2e H2D), read through self.c by the step
        self.cidx = {m: i for i, m in enumerate(need)}
        self.perm = torch.empty(n, dtype=torch.int32, device=dev)
        ne.ne_gen_perm_i32(self.seed, 6, self.perm)
        self.v = torch.empty(self.B, dtype=torch.int32, device=dev)
        ne.ne_gen_uniform_i32(self.seed, 7, 0, -self.vr, self.vr, self.v)
        self.eps_s = {m: torch.empty(n, dtype=torch.int64, device=dev) for m in self.owned}
        self.pay = [torch.empty(hi - lo, dtype=torch.int64, device=dev) for _, lo, hi in self.items]
        self.b0, b1 = part_range(self.nb, world, rank, 32)
        nc = b1 - self.b0
        self.delta = [torch.zeros(nc, dtype=torch.int64, device=dev) for _ in range(M)]
        self.dout = [torch.empty(nc, dtype=torch.int64, device=dev) for _ in range(M)]
        self.drec = [torch.empty(nc, dtype=torch.int64, device=dev) for _ in range(M)]
        self.bitmap = torch.empty((nc + 31) // 32, dtype=torch.int32, device=dev)
        self.diag = ne.diag_new()
        self.partitioned, self.has_collective = True, True
        self.placement = True
        self.launches_per_step = len(self.owned) + len(self.items) + 2
        self.partition_note = (f"stream placement: rank {rank} of {world} entangles stream(s) {self.owned} and gathers "
                               f"+ inner-products block range(s) {[(m, lo, hi) for m, lo, hi in self.items]}; "
                               f"all_gather of the M x {self.nb} block sums; checks/recovers blocks "
                               f"[{self.b0}, {b1})")

    def _placement_stages(self, i):
        from paper_1604_04740_b200.dist import c4_allgather

        ne, cfg, M, B = self.ne, self.cfg, self.M, self.B
        r = i % M
        nc = self.dout[0].numel()

        def entangle():
            for m in self.owned:
                ne.ne_entangle_stream(cfg, m, self.c[self.cidx[m]], self.c[self.cidx[(m - 1) % M]], self.eps_s[m],
                                      self.diag)

        def gather_inner():
            for (m, lo, hi), out in zip(self.items, self.pay):
                ne.ne_op_permute_inner_stream(cfg, self.eps_s[m], self.perm, self.v, B, lo, hi - lo, out)

        def exchange():
            full = c4_allgather(self.pay, M, self.nb)
            self.delta = [t[self.b0:self.b0 + nc] for t in full]

        return [("entangle", entangle), ("permute_inner", gather_inner), ("allgather", exchange),
                ("check", lambda: ne.ne_disentangle_check(cfg, self.delta, 0, self.dout, self.bitmap, self.diag)),
                ("recover", lambda: ne.ne_recover(cfg, [None if m == r else self.delta[m] for m in range(M)], r,
                                                  self.drec))]

    def stages(self, i):
        if getattr(self, "placement", False):
            return self._placement_stages(i)
        ne, cfg = self.ne, self.cfg
        r = i % 4
        part = [None if m == r else self.delta[m] for m in range(4)]
        if self.w == 32:
            return [
                ("entangle", lambda: ne.ne_entangle_aos_w32(cfg, self.c, self.eps, self.diag)),
                ("permute_inner_check", lambda: ne.ne_op_permute_inner_check_w32(
                    cfg, self.eps, self.v, self.B, 0, self.dout, perm=self.perm, delta_out=self.delta,
                    bitmap=self.bitmap, diag=self.diag)),
                ("recover", lambda: ne.ne_recover_w32(cfg, part, r, self.drec)),
            ]
        if self.layout != "aos":
            return [
                ("entangle", lambda: ne.ne_entangle(cfg, self.c, self.eps, self.diag)),
                ("permute_inner_check", lambda: ne.ne_op_permute_inner_check(
                    cfg, self.v, self.B, 0, self.dout, x=self.eps, perm=self.perm, n=self.n,
                    delta_out=self.delta, bitmap=self.bitmap, diag=self.diag)),
                ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec)),
            ]
        if self.algo == "bucket":
            return [
                ("entangle", lambda: ne.ne_entangle_aos(cfg, self.c, self.eps, self.diag)),
                ("permute_inner_check", lambda: ne.ne_op_permute_inner_check_bucketed(
                    cfg, self.eps, self.perm, self.v, self.B, 0, self.delta, self.dout, self.ws,
                    self.bitmap, self.diag)),
                ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec)),
            ]
        return [
            ("entangle", lambda: ne.ne_entangle_aos(cfg, self.c, self.eps, self.diag)),
            ("permute_inner_check", lambda: ne.ne_op_permute_inner_check(
                cfg, self.v, self.B, 0, self.dout, x_aos=self.eps, perm=self.perm, n=self.n,
                delta_out=self.delta, bitmap=self.bitmap, diag=self.diag)),
            ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec)),
        ]

    def work_per_step(self):  # algorithmic GB per step: entangle 48 B + gather/inner 36 B per position (w = 64)
        if self.w == 32:      # entangle 16 + 16 B, gather 16 B + 4 B index
            return self.n * (32 + 20) / 1e9
        return self.n * (48 + 36) / 1e9

    def global_work(self):  # the whole C4 problem's algorithmic bytes (the single-GPU AoS accounting)
        return self.n * (48 + 36) / 1e9

    def extra_roofline(self, dom, ms, peaks):
        """The gather's own floor (profiles/r02_c4_floor.md): every random
        32-B sector read costs one 128-B DRAM line fill on B200 (4 sectors per
        L2 request, unchanged by any cache hint or fetch-granularity limit),
        so the fused gather + inner + check moves >= 128 B + its 4-B index per
        gathered position."""
        if dom != "permute_inner_check" or self.layout != "aos" or getattr(self, "placement", False):
            return None
        if self.algo == "bucket":   # what the scatter-reduce moves per position (ne_permute_inner_plan)
            plan = self.ne.ne_permute_inner_plan(self.cfg, self.n, self.B)
            if plan["mode"] == 1:   # perm 4 + 32-bit pairs written and read 4 + 4 + eps 32 + run index written and read
                per = 44 + 2 * plan["index_bytes"] / self.n
                how = ("owned-run scatter-reduce: perm read, 32-bit pairs written and read, the run index written "
                       "and read, every eps entry read once from its window (L2-resident while its cells are reduced)")
            else:                   # perm 4 + 8-byte pairs written and read 8 + 8 + eps 32
                per = 52
                how = ("bucketed scatter-reduce: perm read, (i, perm[i]) pairs written and read, every eps entry "
                       "read once from its window (L2-resident while its bucket is consumed)")
            gb = self.n * per / 1e9
            ach = gb / (ms / 1e3)
            return {"bytes_per_position": round(per, 3), "bytes_per_launch_GB": round(gb, 3), "achieved": round(ach, 1),
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
                    "floor_ms": round(gb / peaks["hbm_gbs"] * 1e3, 3), "plan": plan, "evidence": how}
        per = 128 + 4
        gb = self.n * per / 1e9
        ach = gb / (ms / 1e3)
        return {"bytes_per_position": per, "bytes_per_launch_GB": round(gb, 3), "achieved": round(ach, 1),
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
                "floor_ms": round(gb / peaks["hbm_gbs"] * 1e3, 3),
                "evidence": "profiles/r02_c4_floor.md (ncu: 4 DRAM sectors per random 32-B load)"}

    def stage_info(self):
        n, nb = self.n, self.nb
        if getattr(self, "placement", False):
            npos = sum(hi - lo for _, lo, hi in self.items) * self.B
            nc = self.dout[0].numel()
            return {"entangle": ("hbm", len(self.owned) * n * 16 / 1e9, "GB"),
                    "permute_inner": ("hbm", npos * 12 / 1e9, "GB"),
                    "allgather": ("nvlink", self.M * nb * 8 / 1e9, "GB"),
                    "check": ("hbm", nc * self.M * 16 / 1e9, "GB"),
                    "recover": ("hbm", nc * 7 * 8 / 1e9, "GB")}
        if self.w == 32:
            return {"entangle": ("hbm", n * 32 / 1e9, "GB"),
                    "permute_inner_check": ("hbm", (n * 20 + nb * 4 * 8) / 1e9, "GB"),
                    "recover": ("hbm", nb * 7 * 4 / 1e9, "GB")}
        return {"entangle": ("hbm", n * 48 / 1e9, "GB"),
                "permute_inner_check": ("hbm", (n * 36 + nb * 4 * 16) / 1e9, "GB"),
                "recover": ("hbm", nb * 7 * 8 / 1e9, "GB")}

    def config(self):
        wl = ("C4 (BASELINE configs[3]): M=4 streams of 2^28 int32 U[-2^12,2^12), seeded "
              "permutation, inner products with a shared 1024-vector in blocks of 1024")
        if self.w == 32:
            wl = ("C4 shape at w = 32 (NEXT-3): M=4 streams of 2^28 int32 U[-64,64) (C4's U[-2^12,2^12) "
                  "does not fit 32-bit containers), seeded permutation, 1024-blocked inner products with a "
                  "shared U[-64,64) vector")
        return {"workload": wl,
                "M": 4, "n": self.n, "block": self.B,
                "layout": ("AoS (position-major) entangled int32 (16 B per position)" if self.w == 32 else
                           "AoS (position-major) entangled int64" if self.layout == "aos" else
                           "SoA (one int64 stream per m; 4 random sectors per gathered position)"),
                "entanglement": {"l": self.cfg.l, "k": self.cfg.k, "w": self.w},
                "l2": "working set ~13 GB >> 126 MB L2 (no flush needed)",
                "step": ("entangle(AoS)+bucketed scatter-reduce permute/inner + disentangle/check(r=0)"
                         "+recover(r=step mod 4)" if self.algo == "bucket" else
                         "entangle(AoS)+gather/inner/disentangle/check fused(r=0)+recover(r=step mod 4)"),
                "c4algo": self.algo}

    def plain_times(self, reps=3):
        """Same gather + inner kernel on plain (unentangled) data in the same
        int64 AoS containers, no check: the paper's conventional routine."""
        torch, ne = self.torch, self.ne
        if self.layout != "aos" or self.w != 64 or getattr(self, "placement", False):
            return {}
        plain = torch.stack([x.to(torch.int64) for x in self.c], dim=1).reshape(-1).contiguous()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if self.algo == "bucket":
            run = lambda: ne.ne_op_permute_inner_check_bucketed(  # noqa: E731
                self.cfg, plain, self.perm, self.v, self.B, 0, self.delta, self.drec, self.ws)
            what = ("partitioned scatter-reduce + inner (+check, meaningless on plain data) on plain int64 AoS "
                    "containers, inputs already widened")
        else:
            run = lambda: ne.ne_op_permute_inner_check(  # noqa: E731
                self.cfg, self.v, self.B, 0, self.drec, x_aos=plain, perm=self.perm, n=self.n, delta_out=self.delta)
            what = ("gather+inner (+check, skipped on plain data) on plain int64 AoS containers, "
                    "inputs already widened")
        run()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        del plain
        return {"plain_same_kernel": (e0.elapsed_time(e1) / reps, what)}

    def oracle_sample(self, blocks):
        import oracle as O

        ocfg = O.config_for(4, self.w)
        n, B, vr = self.n, self.B, self.vr
        t0 = time.perf_counter()
        idx = O.gen_perm(self.seed, 6, n, blocks * B, self.b0 * B)
        v = O.gen_uniform(self.seed, 7, 0, -vr, vr, B)
        c = np.stack([np.concatenate([O.gen_uniform(self.seed, 1, m, -vr, vr, 1, int(p)) for p in idx])
                      for m in range(4)])
        eps = O.entangle(ocfg, c)
        delta = O.op_inner(ocfg, eps, v, B)
        d, _, _ = O.disentangle_check(ocfg, delta, 0)
        dt = time.perf_counter() - t0
        self._oref = (delta, d)
        return dt, blocks * B * (84 if self.w == 64 else 52) / 1e9, \
            f"{blocks} output blocks of 1024 gathered positions (of {n // B})"

    def oracle_compare(self):
        if getattr(self, "_oref", None) is None:
            return None
        D, d = self._oref
        nb = D.shape[1]
        got_d = np.stack([t[:nb].to(self.torch.int64).cpu().numpy() for t in self.delta])
        got = np.stack([t[:nb].to(self.torch.int64).cpu().numpy() for t in self.dout])
        return bool((got_d == D).all() and (got == d).all())


class C2Conv(Workload):
    # the Toeplitz tap matrix does not depend on the entangle (or ABFT's encode), nor the recovery on the check
    concurrent = {"prep_g": ("entangle", "encode"), "recover": "check"}
    """configs[1]: M=3 streams of 65536 int32 U[-128,128), circular convolution
    with a shared 64-tap kernel U[-128,128), entangled int64.  algo "tc": the
    Toeplitz GEMM on tcgen05 over extended digit planes (k_conv_tc.cu);
    "direct": the IMAD kernel (k_conv.cu).  The paper's own conv shape
    (P:1106-1108: N_in = 10^6, 100-4500 taps, M in {3, 8}) is workload c2p."""

    name = "C2"
    metric_unit = "Gop/s"
    E2E_IN = ("c", "g")
    E2E_OUT = ("dout",)

    def __init__(self, rank, n=65536, taps=64, seed=1, M=3, algo="tc", paper=False, fuse=True, scheme="entangled",
                 world=1, scaling="strong"):
        import torch
        import paper_1604_04740_b200 as ne
        from paper_1604_04740_b200.dist import HALO, part_range

        self.ne, self.torch = ne, torch
        self.M, self.n, self.T, self.algo, self.paper = M, n, taps, algo, paper
        self.scheme = scheme if algo == "tc" else "entangled"
        self.fuse = fuse and algo == "direct"  # the direct conv kernel carries the fused check
        if paper:
            self.name = "C2P"
        if scaling == "strong" and world > 1 and not (algo == "direct" and self.fuse and taps - 1 <= HALO):
            scaling = "weak"   # only the direct fused conv has the halo partition; the others run replicas
            self.partition_note = "replicas (the halo partition exists for the direct fused conv only)"
        self.seed = self.setup_partition(rank, world, scaling, seed)
        self.n_global, self.lo, self.halo = n, 0, 0
        if self.partitioned:
            # contiguous position ranges + a circular halo of HALO >= T - 1 positions from rank - 1
            self.lo, hi = part_range(n, world, rank, 32)
            self.n = n = hi - self.lo
            self.halo = HALO
            self.has_collective = True
            self.partition_note = (f"positions [{self.lo}, {hi}) of all M streams on rank {rank} of {world}, plus a "
                                   f"halo of the previous rank's last {HALO} entangled positions per stream "
                                   f"(send/recv, {HALO * M * 8} B per rank and step); the conv runs over the "
                                   f"extended range and its own positions are exact (T - 1 = {taps - 1} <= {HALO})")
        self.cfg = ne.ne_config_for(M)
        self.c = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(M)]
        for m in range(M):
            ne.ne_gen_uniform_i32(self.seed, 1, m, -128, 128, self.c[m], self.lo)
        self.g = torch.empty(taps, dtype=torch.int32, device="cuda")
        ne.ne_gen_uniform_i32(self.seed, 3, 0, -128, 128, self.g)
        H = self.halo
        mk = lambda: [torch.empty(H + n, dtype=torch.int64, device="cuda") for _ in range(M)]  # noqa: E731
        if H:
            # extended buffers: [halo | own positions]; the own part starts 8 H = 512 B in (16-B aligned)
            self.eps_ext, self.delta_ext, self.dout_ext = mk(), mk(), mk()
            self.delta = [t[H:] for t in self.delta_ext]
            self.dout = [t[H:] for t in self.dout_ext]
            self.drec = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(M)]
            self.E2E_OUT = ("dout_ext",)
        else:
            self.delta, self.dout, self.drec = mk(), mk(), mk()
        if algo == "tc":
            # c in [-128, 127] (U[-128, 128)): exactly the int8 range, so eps = c_m + 2^l c_{m-1}
            # is its two int8 halves (the pair plan; |c| <= 127 in the plan's symmetric terms
            # plus c = -128, whose digit is still int8); the entangle kernel asserts it per value
            self.L, self.limb_bits = ne.ne_gemm_limb_plan(self.cfg, 127)
            self.block, self.kpad, self.plen = ne.ne_conv_geometry(n, taps, self.L)
            self.planes = torch.empty(M * self.L * self.plen, dtype=torch.int8, device="cuda")
            if self.scheme == "abft":
                # the paper's comparison: plain data (one int8 digit per stream) + the checksum
                # stream (Eq. 4; |sum| <= 128 M -> 2 base-256 digits)
                self.Ls = 2
                self.pdata = torch.empty(M * self.plen, dtype=torch.int8, device="cuda")
                self.psum = torch.empty(self.Ls * self.plen, dtype=torch.int8, device="cuda")
                self.e = torch.empty(n, dtype=torch.int64, device="cuda")
            self.Gt = torch.empty(self.block * self.kpad, dtype=torch.int8, device="cuda")
            self.launches_per_step = 5 + (1 if n % 128 else 0)
        elif H:
            self.launches_per_step = 3   # + the halo send/recv (NCCL)
        else:
            self.eps = mk()
            self.launches_per_step = 3 if self.fuse else 4
        self.bitmap = torch.empty((H + n + 31) // 32, dtype=torch.int32, device="cuda")
        self.diag = ne.diag_new()

    def stages(self, i):
        ne, cfg, M = self.ne, self.cfg, self.M
        r = i % M
        part = [None if m == r else self.delta[m] for m in range(M)]
        tail = [("check", lambda: ne.ne_disentangle_check(cfg, self.delta, 0, self.dout, self.bitmap, self.diag)),
                ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec))]
        if self.scheme == "abft":
            rr = [None if m == r else self.delta[m] for m in range(M)]
            return [("encode", lambda: ne.ne_abft_encode_conv(cfg, self.c, self.T, 0, self.block, self.pdata, self.Ls,
                                                              self.psum, self.diag)),
                    ("prep_g", lambda: ne.ne_conv_prep_taps(self.g, 0, self.Gt, self.diag, self.block)),
                    ("conv", lambda: (ne.ne_op_conv_limbs_plain(M, self.pdata, 1, self.Gt, self.n, self.T, 0,
                                                                self.delta, block=self.block),
                                      ne.ne_op_conv_limbs_plain(1, self.psum, self.Ls, self.Gt, self.n, self.T, 0,
                                                                [self.e], block=self.block))),
                    ("check", lambda: ne.ne_abft_check(cfg, self.delta, self.e, self.bitmap, self.diag)),
                    ("recover", lambda: ne.ne_abft_recover(cfg, rr, self.e, r, self.drec[r]))]
        if self.algo == "tc":
            return [("entangle", lambda: ne.ne_entangle_limbs_conv(cfg, self.c, self.T, 0, self.L, self.planes,
                                                                   self.diag, self.limb_bits, self.block)),
                    ("prep_g", lambda: ne.ne_conv_prep_taps(self.g, 0, self.Gt, self.diag, self.block)),
                    ("conv", lambda: ne.ne_op_conv_limbs(cfg, self.planes, self.L, self.Gt, self.n, self.T, 0,
                                                         self.delta, self.limb_bits, self.block))] + tail
        if self.halo:
            from paper_1604_04740_b200.dist import halo_exchange

            H = self.halo
            return [("entangle", lambda: ne.ne_entangle(cfg, self.c, [t[H:] for t in self.eps_ext], self.diag)),
                    ("halo", lambda: halo_exchange(self.eps_ext, H, self.n)),
                    ("conv_check", lambda: ne.ne_op_conv_check(cfg, self.eps_ext, self.g, self.delta_ext, 0,
                                                               self.dout_ext, self.bitmap, self.diag)),
                    tail[1]]
        if self.fuse:
            return [("entangle", lambda: ne.ne_entangle(cfg, self.c, self.eps, self.diag)),
                    ("conv_check", lambda: ne.ne_op_conv_check(cfg, self.eps, self.g, self.delta, 0, self.dout,
                                                               self.bitmap, self.diag)),
                    tail[1]]
        return [("entangle", lambda: ne.ne_entangle(cfg, self.c, self.eps, self.diag)),
                ("conv", lambda: ne.ne_op_conv(cfg, self.eps, self.g, self.delta))] + tail

    def work_per_step(self):
        return 2 * self.M * self.n * self.T / 1e9

    def global_work(self):
        return 2 * self.M * self.n_global * self.T / 1e9

    def stage_info(self):
        n, M, T = self.n, self.M, self.T
        info = {"check": ("hbm", M * n * 16 / 1e9, "GB"),
                "recover": ("hbm", (2 * M - 1) * n * 8 / 1e9, "GB")}
        if self.scheme == "abft":
            info["conv"] = ("tensor", 2 * (M + self.Ls) * n * T / 1e12, "TOP")
            info["encode"] = ("hbm", (M * n * 4 + (M + self.Ls) * self.plen) / 1e9, "GB")
            info["prep_g"] = ("hbm", (T * 4 + self.block * self.kpad) / 1e9, "GB")
            info["check"] = ("hbm", (M + 1) * n * 8 / 1e9, "GB")
            info["recover"] = ("hbm", (M + 1) * n * 8 / 1e9, "GB")
        elif self.algo == "tc":
            # useful limb products only (the Toeplitz zeros, Kpad/T - 1, are not counted)
            info["conv"] = ("tensor", 2 * self.L * M * n * T / 1e12, "TOP")
            info["entangle"] = ("hbm", M * (n * 4 + self.L * self.plen) / 1e9, "GB")
            info["prep_g"] = ("hbm", (T * 4 + self.block * self.kpad) / 1e9, "GB")
        else:
            info["conv"] = ("alu", M * n * T / 1e12, "TMAC")
            info["conv_check"] = ("alu", M * n * T / 1e12, "TMAC")
            info["entangle"] = ("hbm", M * n * 12 / 1e9, "GB")
        return info

    def config(self):
        if self.paper:
            wl = (f"C2P (the paper's convolution shape, P:1106-1108): M={self.M} streams of N_in={self.n} int32 "
                  f"U[-128,128), circular convolution with a {self.T}-tap kernel U[-128,128)")
        else:
            wl = ("C2 (BASELINE configs[1]): M=3 streams of 65536 int32 U[-128,128), circular "
                  "convolution with a shared 64-tap kernel U[-128,128)")
        ws = self.M * self.n * 8 * 3 / 1e6
        if self.scheme == "abft":
            wl += "; scheme: ABFT single checksum stream (Eqs. 3-6, the paper's comparison method)"
        return {"workload": wl, "M": self.M, "n": self.n, "taps": self.T, "scheme": self.scheme,
                "conv_algo": ("tc: Toeplitz GEMM on tcgen05, %d int8 digits base 2^%d, %d-output blocks, Kpad=%d"
                              % (self.L, self.limb_bits, self.block, self.kpad)) if self.algo == "tc" else "direct IMAD",
                "entanglement": {"l": self.cfg.l, "k": self.cfg.k, "w": 64},
                "l2": (f"working set {ws:.0f} MB" + (" fits L2 (launch-latency bound)" if ws < 100 else " > L2")),
                "step": "entangle+prep_taps+conv+disentangle/check(r=0)+recover(r=step mod M)"
                if self.algo == "tc" else ("entangle+conv with fused disentangle/check(r=0)+recover(r=step mod M)"
                                           if self.fuse else
                                           "entangle+conv+disentangle/check(r=0)+recover(r=step mod M)")}

    def plain_times(self, reps=20):
        """The same conv kernel on unentangled data: (i) same digit count
        (plain c in digit 0, other digits 0), (ii) one int8 digit; ms per call."""
        torch, ne = self.torch, self.ne
        if self.scheme == "abft":
            return {}
        if self.algo != "tc":
            x64 = [c.to(torch.int64) for c in self.c]
            o64 = [torch.empty_like(x) for x in x64]
            return {"plain_same_kernel": (self._time(lambda: ne.ne_op_conv(self.cfg, x64, self.g, o64), reps),
                                          "direct conv kernel on plain int64 streams, inputs already widened")}
        M, out = self.M, {}
        for tag, L in (("plain_same_kernel", self.L), ("plain_native_L1", 1)):
            planes = torch.zeros(M * L * self.plen, dtype=torch.int8, device="cuda")
            pv = planes.view(M, L, self.plen)
            s0 = self.T - 1
            idx = (torch.arange(self.plen, device="cuda") - s0) % self.n  # same extended layout
            for m in range(M):
                pv[m, 0].copy_(self.c[m][idx].to(torch.int8))
            ne.ne_op_conv_limbs(self.cfg, planes, L, self.Gt, self.n, self.T, 0, self.delta, self.limb_bits, self.block)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                ne.ne_op_conv_limbs(self.cfg, planes, L, self.Gt, self.n, self.T, 0, self.delta, self.limb_bits,
                                    self.block)
            e1.record()
            torch.cuda.synchronize()
            out[tag] = (e0.elapsed_time(e1) / reps, f"Toeplitz conv GEMM (L={L}) on plain digit planes (planes "
                                                    f"prepared outside the timing)")
            del planes
        return out

    def oracle_sample(self, reps):
        import oracle as O

        M = self.M
        ocfg = O.config_for(M, 64)
        c = np.stack([O.gen_uniform(self.seed, 1, m, -128, 128, self.n_global) for m in range(M)])
        g = O.gen_uniform(self.seed, 3, 0, -128, 128, self.T)
        if self.paper:
            # bounded sample: the same pipeline at N' = 16384 (same M, taps, distributions)
            n2 = 16384
            c = np.stack([O.gen_uniform(self.seed, 1, m, -128, 128, n2) for m in range(M)])
            t0 = time.perf_counter()
            eps = O.entangle(ocfg, c)
            d = O.op_conv(ocfg, eps, g)
            dh, _, _ = O.disentangle_check(ocfg, d, 0)
            dt = time.perf_counter() - t0
            # positions T-1 .. N'-1 of the N' prefix never wrap: they equal the full-size outputs
            self._oref = (self.T - 1, d[:, self.T - 1:], dh[:, self.T - 1:])
            return dt, 2 * M * n2 * self.T / 1e9, f"one full pass at N'={n2} (M={M}, T={self.T}, same distributions)"
        t0 = time.perf_counter()
        for _ in range(reps):
            eps = O.entangle(ocfg, c)
            d = O.op_conv(ocfg, eps, g)
            dh, _, _ = O.disentangle_check(ocfg, d, 0)
        dt = time.perf_counter() - t0
        a, b = self.lo, self.lo + self.n   # this rank's positions (all of them on one GPU)
        self._oref = (a, d[:, a:b], dh[:, a:b])
        return dt, reps * self.global_work(), f"{reps} full C2 passes"

    def oracle_compare(self):
        if getattr(self, "_oref", None) is None or self.scheme != "entangled":
            return None
        glo, D, d = self._oref   # global position of the first compared output
        lo = glo - self.lo
        hi = lo + D.shape[1]
        got_d = np.stack([t[lo:hi].cpu().numpy() for t in self.delta])
        got = np.stack([t[lo:hi].cpu().numpy() for t in self.dout])
        return bool((got_d == D).all() and (got == d).all())


class C1Chain(Workload):
    """configs[0]: M=3 streams of 4096 int32 U[-2^10,2^10), seed 0; scale by 37
    then add a second seeded 3-stream set; disentangle + check.  w = 64
    containers (default) or the paper's w = 32 instantiation (l = 11, k = 10,
    P:528-530; range +-1 046 528 admits C1's bound 38 912).  --n sweeps the
    stream length (HBM-bound from ~2^20 on)."""

    name = "C1"
    metric_unit = "Gpositions/s"
    E2E_IN = ("c", "a")
    E2E_OUT = ("dout",)

    def __init__(self, rank, n=4096, seed=0, w=64, fuse=True, world=1, scaling="strong"):
        import torch
        import paper_1604_04740_b200 as ne
        from paper_1604_04740_b200.dist import part_range

        self.ne, self.torch = ne, torch
        self.M, self.n, self.w, self.fuse = 3, n, w, fuse
        if (n, w) != (4096, 64):
            self.name = f"C1_w{w}_n{n}"  # traffic.json key of the sweep lines
        self.seed = self.setup_partition(rank, world, scaling, seed)
        self.n_global, self.lo = n, 0
        if self.partitioned:
            # contiguous position ranges, all M streams of a range on this rank (whole bitmap words)
            self.lo, hi = part_range(n, world, rank, 32)
            self.n = n = hi - self.lo
            self.partition_note = (f"positions [{self.lo}, {hi}) of all M streams on rank {rank} of {world}; "
                                   "a1-a5 local, counters all-reduced after the step")
        self.cfg = ne.ne_config_for(3, w)
        dt = torch.int64 if w == 64 else torch.int32
        mk32 = lambda: [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(3)]  # noqa: E731
        mk = lambda: [torch.empty(n, dtype=dt, device="cuda") for _ in range(3)]  # noqa: E731
        self.c, self.a = mk32(), mk32()
        for m in range(3):
            ne.ne_gen_uniform_i32(self.seed, 1, m, -1024, 1024, self.c[m], self.lo)
            ne.ne_gen_uniform_i32(self.seed, 2, m, -1024, 1024, self.a[m], self.lo)
        self.eps, self.alpha, self.dout, self.drec = mk(), mk(), mk(), mk()
        self.bitmap = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        self.diag = ne.diag_new()
        # fused: entangle_sets (1 launch; 2 for w = 64 streams > 2^22) + op/check + recover
        self.launches_per_step = (3 if (w == 32 or n <= (1 << 22)) else 4) if fuse else 5

    def stages(self, i):
        ne, cfg = self.ne, self.cfg
        r = i % 3
        part = [None if m == r else self.eps[m] for m in range(3)]
        if self.fuse:
            # operand set c and addend set a entangled in one launch (two stream sets)
            if self.w == 32:
                ent = lambda: ne.ne_entangle_sets_w32(cfg, self.c + self.a, 2, self.eps + self.alpha,  # noqa: E731
                                                      self.diag)
                opc = lambda: ne.ne_op_scale_add_check_w32(cfg, self.eps, 37, self.alpha, 0, self.dout,  # noqa: E731
                                                           self.bitmap, self.diag)
                rec = lambda: ne.ne_recover_w32(cfg, part, r, self.drec)  # noqa: E731
            else:
                ent = lambda: ne.ne_entangle_sets(cfg, self.c + self.a, 2, self.eps + self.alpha,  # noqa: E731
                                                  self.diag)
                opc = lambda: ne.ne_op_scale_add_check(cfg, self.eps, 37, self.alpha, 0, self.dout,  # noqa: E731
                                                       self.bitmap, self.diag)
                rec = lambda: ne.ne_recover(cfg, part, r, self.drec)  # noqa: E731
            return [("entangle", ent), ("scale_add_check", opc), ("recover", rec)]
        if self.w == 32:
            return [("entangle", lambda: (ne.ne_entangle_w32(cfg, self.c, self.eps, self.diag),
                                          ne.ne_entangle_w32(cfg, self.a, self.alpha, self.diag))),
                    ("scale_add", lambda: ne.ne_op_scale_add_w32(cfg, self.eps, 37, None, self.alpha, 1)),
                    ("check", lambda: ne.ne_disentangle_check_w32(cfg, self.eps, 0, self.dout, self.bitmap,
                                                                  self.diag)),
                    ("recover", lambda: ne.ne_recover_w32(cfg, part, r, self.drec))]
        return [("entangle", lambda: (ne.ne_entangle(cfg, self.c, self.eps, self.diag),
                                      ne.ne_entangle(cfg, self.a, self.alpha, self.diag))),
                ("scale_add", lambda: ne.ne_op_scale_add(cfg, self.eps, 37, self.alpha)),
                ("check", lambda: ne.ne_disentangle_check(cfg, self.eps, 0, self.dout, self.bitmap, self.diag)),
                ("recover", lambda: ne.ne_recover(cfg, part, r, self.drec))]

    def work_per_step(self):
        return self.n / 1e9

    def global_work(self):
        return self.n_global / 1e9

    def stage_info(self):
        n, B = self.n, self.w // 8
        sa = 3 * n * 3 * B  # fused scale + add: read eps, alpha, write eps
        return {"entangle": ("hbm", 2 * 3 * n * (4 + B) / 1e9, "GB"), "scale_add": ("hbm", sa / 1e9, "GB"),
                "scale_add_check": ("hbm", (sa + 3 * n * B + n / 8) / 1e9, "GB"),  # + d_hat written
                "check": ("hbm", 3 * n * 2 * B / 1e9, "GB"), "recover": ("hbm", 5 * n * B / 1e9, "GB")}

    def config(self):
        small = self.n * 3 * 4 * 2 < 100e6
        return {"workload": "C1 (BASELINE configs[0]): M=3 streams of %d int32 U[-2^10,2^10), seed 0; "
                            "scale by 37, add a second seeded 3-stream set; disentangle+check" % self.n,
                "M": 3, "n": self.n, "w": self.w, "entanglement": {"l": self.cfg.l, "k": self.cfg.k, "w": self.w},
                "l2": ("%.1f MB working set (launch-latency bound)" % (self.n * 3 * (8 + 4 * self.w // 8) / 1e6))
                if small else "working set >> 126 MB L2 (no flush needed)",
                "step": "entangle(c, a: one launch) + scale/add with fused disentangle/check(r=0) + "
                        "recover(r=step mod 3)"
                if self.fuse else "entangle(c, a) + scale/add + disentangle/check(r=0) + recover(r=step mod 3)"}

    def plain_times(self, reps=20):
        """The conventional routine on unentangled data (the paper's comparison,
        F5): (i) the same scale+add kernel on plain values in the same
        containers, (ii) the narrowest native form (int32 plain data, the w = 32
        kernel); ms per call.  overhead_pct = step / plain - 1."""
        torch, ne = self.torch, self.ne
        cfg32 = ne.ne_config_for(3, 32)
        x32 = [c.clone() for c in self.c]
        native = (self._time(lambda: ne.ne_op_scale_add_w32(cfg32, x32, 37, None, self.a, 1), reps),
                  "scale+add kernel in place on the plain int32 inputs (w = 32 kernel)")
        if self.w == 32:
            return {"plain_same_kernel": native}
        x64 = [c.to(torch.int64) for c in self.c]
        a64 = [a.to(torch.int64) for a in self.a]
        same = (self._time(lambda: ne.ne_op_scale_add(self.cfg, x64, 37, a64), reps),
                "the same scale+add kernel on plain int64 containers (inputs already widened)")
        return {"plain_same_kernel": same, "plain_native_int32": native}

    def oracle_sample(self, reps):
        import oracle as O

        ocfg = O.config_for(3, self.w)
        ns = min(self.n, 1 << 16)
        c = np.stack([O.gen_uniform(self.seed, 1, m, -1024, 1024, ns, self.lo) for m in range(3)])
        a = np.stack([O.gen_uniform(self.seed, 2, m, -1024, 1024, ns, self.lo) for m in range(3)])
        t0 = time.perf_counter()
        for _ in range(reps):
            d = O.op_add(ocfg, O.op_scale(ocfg, O.entangle(ocfg, c), 37), O.entangle(ocfg, a))
            dh, _, _ = O.disentangle_check(ocfg, d, 0)
        dt = time.perf_counter() - t0
        self._oref = (d, dh)
        return dt, reps * ns / 1e9, f"{reps} full C1 passes (w={self.w})" + ("" if ns == self.n else f" at N'={ns}")

    def oracle_compare(self):
        """delta (left in eps by the in-place op) and d_hat of the timed run vs the oracle."""
        if getattr(self, "_oref", None) is None:
            return None
        D, d = self._oref
        ns = d.shape[1]
        got = np.stack([t[:ns].to(self.torch.int64).cpu().numpy() for t in self.dout])
        got_d = np.stack([t[:ns].to(self.torch.int64).cpu().numpy() for t in self.eps])
        return bool((got == d).all() and (got_d == D).all())


WORKLOADS = {"c1": C1Chain, "c2": C2Conv, "c2p": C2Conv, "c3": C3Gemm, "c3p": C3Gemm, "c4": C4PermInner, "c5": None}
ORACLE_SAMPLE = {"c1": (200, 20), "c2": (20, 2), "c2p": (1, 1), "c3": (16, 2), "c3p": (64, 8), "c4": (64, 8),
                 "c5": (4096, 512)}  # (cpu_baseline, per reference-arm step)


def make_workload(args, rank, world=1):
    kw = dict(world=world, scaling=args.scaling)
    if args.workload == "c3":
        return C3Gemm(rank, algo=args.algo, scheme=args.scheme, limbs=args.limbs, fuse=bool(args.fuse or 0),
                      abound=args.abound, bbound=args.bbound, **kw)
    if args.workload == "c3p":
        return C3Gemm(rank, algo=args.algo, scheme=args.scheme, limbs=args.limbs, fuse=bool(args.fuse or 0),
                      paper_shape=(args.streams, 2000, 1200, args.kdim), **kw)
    if args.workload == "c2":
        return C2Conv(rank, algo=args.conv or "direct", fuse=bool(args.fuse if args.fuse is not None else 1), **kw)
    if args.workload == "c2p":
        return C2Conv(rank, n=10 ** 6, taps=args.taps, M=args.streams, algo=args.conv or "tc", paper=True,
                      scheme=args.scheme, **kw)
    if args.workload == "c4":
        return C4PermInner(rank, layout=args.layout, w=args.w, algo=args.c4algo, **kw)
    if args.workload == "c1":
        return C1Chain(rank, n=args.n or 4096, w=args.w, fuse=bool(args.fuse if args.fuse is not None else 1), **kw)
    return WORKLOADS[args.workload](rank)


METRIC = "entangled LSB Gop/s (or GB/s) at 1/2/4/8 B200, % roofline, % overhead vs plain"


# ====================================================================== clocks
class ClockSampler:
    """SM clock, power and clock-event reasons sampled through NVML every
    `period_s` (default 2 ms) on a background thread while the timed region
    runs, so the record covers the kernels that dominate it (the GEMM of a
    0.6 ms step included); nvidia-smi -lms 20 as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index, period_s=0.002):
        self.index, self.period = index, period_s
        self.rows, self.max_mhz, self.source = [], None, None
        self._stop = None
        self._thr = None

    def start(self):
        import threading

        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            reasons = [(nm, getattr(N, attr, 0)) for nm, attr in self.REASONS]
            getr = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception:  # noqa: BLE001 — no NVML: no clock record
            self.source = "unavailable"
            return
        self.source = f"NVML every {self.period * 1e3:.0f} ms"
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                try:
                    sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                    pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
                    rs = getr(h)
                    self.rows.append((sm, pw, [nm for nm, bit in reasons if bit and rs & bit]))
                except Exception:  # noqa: BLE001
                    pass
                self._stop.wait(self.period)

        self._thr = threading.Thread(target=loop, daemon=True)
        self._thr.start()

    def stop(self):
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "source": self.source}
        loaded = [r for r in self.rows if r[0] > 500] or self.rows
        reasons = sorted({x for r in loaded for x in r[2]})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_min_mhz": min(r[0] for r in loaded),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(loaded),
                "power_w_max": round(max(r[1] for r in loaded), 1), "source": self.source}


# ====================================================================== runs
def c5_oracle_sample(plan, ncols, keep=None):
    """Row 0 of every stream, the first `ncols` output columns, through the
    oracle: entangle, GEMM, disentangle + check, recovery without plan.kill.
    keep (a dict, optional) receives the oracle's d_hat of those positions."""
    import oracle as O

    M, K, b = plan.M, plan.K, plan.bound
    ocfg = O.config_for(M, 64)
    A0 = np.stack([O.gen_uniform(plan.seed, 4, m, -b, b, K) for m in range(M)])  # row 0 of each block
    B = O.gen_uniform(plan.seed, 5, 0, -b, b, K * plan.cols).reshape(K, plan.cols)[:, :ncols].copy()
    t0 = time.perf_counter()
    E = O.entangle(ocfg, A0)
    D = O.op_gemm(ocfg, E.reshape(M, 1, K), B).reshape(M, -1)
    d, _, _ = O.disentangle_check(ocfg, D, 0)
    O.recover(ocfg, [None if m == (plan.kill or 0) else D[m] for m in range(M)], plan.kill or 0)
    dt = time.perf_counter() - t0
    if keep is not None:
        keep["d"] = d
    return dt, 2 * M * ncols * K / 1e9, f"row 0 of each of the {M} stream blocks, first {ncols} of {plan.cols} columns"


def c5_traffic(streams):
    t = load_traffic()
    g, e = t.get("C5:gemm"), t.get("C5:entangle")
    if not g or not e:
        return None
    return round((g["GB"] + e["GB"]) * streams, 4)


def c5_overhead(be, plan, inp, stage_ms, reps=3):
    """% overhead vs plain for C5 (one GPU, all M streams local): the no-fault
    entangled step (prep_B, entangle + GEMM of every stream, check; the step's
    own stage events) against the plain pipeline of the same scope and launch
    mode (prep_B, then per stream the int32 -> int8 plane and the one-digit
    GEMM: int64 results, and the narrowest native form with int32 products);
    recovery reported as its own cost."""
    import torch

    ne = be.ne
    rows, cols, K, M = plan.rows, plan.cols, plan.K, plan.M
    dev = torch.device("cuda")
    plane = torch.empty(rows * K, dtype=torch.int8, device=dev)
    Bt = torch.empty(cols * K, dtype=torch.int8, device=dev)
    o64 = torch.empty(rows * cols, dtype=torch.int64, device=dev)
    o32 = torch.empty(rows * cols, dtype=torch.int32, device=dev)

    def run(kind):
        ne.ne_gemm_prep_b(inp["B"], K, cols, Bt)
        for m in range(M):
            ne.ne_to_limbs([inp["A"][m][0]], 1, plane)
            if kind == "L1_int64_out":
                ne.ne_op_gemm_limbs_stream(be.cfg, plane, 1, Bt, rows, cols, K, o64, 8)
            else:
                ne.ne_op_gemm_plain_i32(plane, Bt, rows, cols, K, [o32])

    plain = {}
    for kind, scope in (("L1_int64_out", "prep_B + M x (int32 -> int8 plane + one-digit pair GEMM, int64 out)"),
                        ("native_L1", "prep_B + M x (int32 -> int8 plane + one-digit pair GEMM, int32 products)")):
        run(kind)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run(kind)
        e1.record()
        torch.cuda.synchronize()
        plain[kind] = (e0.elapsed_time(e1) / reps, scope)
    nf_keys = [k for k in stage_ms if k in ("entangle_gemm", "exchange", "check", "exchange_check")]
    nf = sum(stage_ms[k] for k in nf_keys)
    rec = stage_ms.get("exchange_recover", 0.0)
    pct = {f"nofault_vs_plain_{k}": round((nf / ms - 1) * 100, 2) for k, (ms, _) in plain.items()}
    pct["failstop_recover_vs_nofault"] = round(rec / nf * 100, 2)
    return {"entangled_nofault": {"ms": round(nf, 4), "scope": "prep_B + M x (entangle + GEMM) + check "
                                                                  "(the timed step's stage events: " + "+".join(nf_keys) + ")"},
            "failstop_recover": {"ms": round(rec, 4), "scope": "recover (stream plan.kill lost)"},
            "plain": {k: {"ms": round(ms, 4), "scope": sc} for k, (ms, sc) in plain.items()},
            "pct": pct,
            "timing": f"eager launches on both sides (as the C5 step), {reps} back-to-back plain pipelines (CUDA events)"}


def run_c5(args, rank, world, local_rank):
    """configs[4]: M = 8 entangled streams (one per GPU when N = 8; stream m on
    rank m mod N otherwise), GEMM 16384^3 int32 U[-32,32) rows sharded, position-
    major all_to_all + check, kill stream 3, survivors recover (NCCL)."""
    import torch
    import torch.distributed as dist

    from paper_1604_04740_b200.dist import (C5Plan, GpuBackend, c5_setup, c5_step, c5_step_failstop,
                                            fused_exchange_ok, make_survivor_groups, owned_streams)

    torch.cuda.set_device(local_rank)
    plan = C5Plan()
    be = GpuBackend(plan.M, plan.bound)
    groups = make_survivor_groups(world, plan.M)
    inp = c5_setup(be, plan)
    # exchange: the GEMM epilogue stores each row block into its owner's
    # symmetric-memory window (fused) when there is something to exchange
    exchange = args.exchange
    if exchange == "auto":
        exchange = "fused" if world > 1 and fused_exchange_ok(plan, world) else "nccl"
    exchange_note = None
    if exchange == "fused":
        try:
            c5_step(be, plan, inp, groups, exchange="fused")
            be.stage_ms()
        except Exception as e:  # symmetric memory unavailable: the all_to_all path (still NCCL over NVLink)
            if args.exchange == "fused":
                raise
            exchange, exchange_note = "nccl", f"fused exchange unavailable ({type(e).__name__}: {e})"[:200]
    for _ in range(args.warmup):
        c5_step(be, plan, inp, groups, exchange=exchange)
        be.stage_ms()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stage_tot, ok, flagged = {}, True, 0
    clk = ClockSampler(local_rank)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        res = c5_step(be, plan, inp, groups, verify=False, exchange=exchange)
        flagged += res["flagged"]
    e1.record()
    torch.cuda.synchronize()
    clk.stop()
    for k, v in be.stage_ms().items():
        stage_tot[k] = stage_tot.get(k, 0.0) + v
    # untimed verification step: recovered outputs == checked outputs (checksums)
    res = c5_step(be, plan, inp, groups, verify=True, exchange=exchange)
    be.stage_ms()
    ok = res.get("checksum_ok") in (True, None)
    total_ms = e0.elapsed_time(e1)
    mine = owned_streams(plan.M, world, rank)

    # end to end: the step's inputs (this rank's A_m, A_{m-1} and B) copied from
    # pinned host memory, its checked outputs copied back, every step
    hA = {m: (a.cpu().pin_memory(), b.cpu().pin_memory()) for m, (a, b) in inp["A"].items()}
    hB = inp["B"].cpu().pin_memory()
    h2d = sum(a.numel() * 4 + b.numel() * 4 for a, b in hA.values()) + hB.numel() * 4
    hout = None
    e2e_steps = max(2, min(args.steps, 5))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for i in range(e2e_steps):
        for m, (a, b) in hA.items():
            inp["A"][m][0].copy_(a, non_blocking=True)
            inp["A"][m][1].copy_(b, non_blocking=True)
        inp["B"].copy_(hB, non_blocking=True)
        r2 = c5_step(be, plan, inp, groups, verify=False, exchange=exchange)
        _, dchk = r2["check_slice"]
        if hout is None:
            hout = [torch.empty(t.numel(), dtype=t.dtype).pin_memory() for t in dchk]
        for h, t in zip(hout, dchk):
            h.copy_(t, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    be.stage_ms()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    d2h = sum(h.numel() * 8 for h in hout)
    if world > 1:
        t = torch.tensor([total_ms, e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0].item()), float(t[1].item())
    ms = total_ms / args.steps

    # real fail-stop (world == M): the rank of stream plan.kill exits its process
    fs = None
    if args.failstop == "exit" and world == plan.M and world > 1:
        be.stage_ms()
        store = dist.distributed_c10d._get_default_store()
        t0 = time.perf_counter()
        rf = c5_step_failstop(be, plan, inp, store, epoch=1, timeout_s=args.failstop_timeout)
        st = be.stage_ms()
        fs = {"real": True, "dead_rank": plan.kill, "view": rf["view"],
              "detect_s_host": round(time.perf_counter() - t0, 3),
              "stages_ms": {k: round(v, 3) for k, v in st.items()},
              "recovered_stream": rf.get("recovered_stream"), "new_world": rf.get("new_world"),
              "reform": rf.get("reform")}
        rank = dist.get_rank()
    if rank != 0:
        return None
    stage_ms = {k: v / args.steps for k, v in stage_tot.items()}
    peaks, peak_src = load_peaks()
    per_rank_streams = len([m for m in range(plan.M) if m % world == rank])
    tops = 2 * be.L * per_rank_streams * plan.rows * plan.cols * plan.K / 1e12
    achieved = tops / (stage_ms["entangle_gemm"] / 1e3)
    peak = peaks["bf16_tflops"] * 2.0
    line = {
        "metric": METRIC, "value": round(2 * plan.M * plan.rows * plan.cols * plan.K / 1e9 / (ms / 1e3), 3),
        "unit": "Gop/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (counter-based splitmix64 generator, gen/ne_gen.h; no dataset)",
        "config": {"workload": "C5 (BASELINE configs[4]): M=8 entangled streams, stream m on rank m mod N; GEMM "
                               "16384x16384x16384 int32 U[-32,32), row block m of A per stream; kill stream 3, "
                               "recover from the other 7",
                   "M": plan.M, "rows_per_stream": plan.rows, "cols": plan.cols, "K": plan.K, "limbs_L": be.L,
                   "kill": plan.kill,
                   "exchange": ("fused: GEMM epilogue TMA-stores each row block into its owner's symmetric-memory "
                                "window (ne_op_gemm_limbs_scatter), device barrier; recovery exchange NCCL "
                                "all_to_all among survivors" if exchange == "fused" else
                                "NCCL all_to_all (torch.distributed)" if world > 1 else
                                "single GPU: all 8 streams local, nothing to exchange")
                   + (f"; {exchange_note}" if exchange_note else "")},
        "roofline": {"bound": "tensor", "kernel": "entangle_gemm (k_entangle_limbs_stream + k_gemm_tc)",
                     "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": "TOP/s",
                     "frac": round(achieved / peak, 4), "traffic": c5_traffic(per_rank_streams),
                     "traffic_unit": "GB per step and rank: ncu DRAM bytes of one stream's entangle + GEMM launch "
                                     "(profiles/traffic.json) x streams on the rank",
                     "peak_source": f"int8 dense = 2 x bf16 burst ({peak_src})"},
        "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        **({"exchange_algbw_GBs": round(len(mine) * plan.rows * plan.cols * 8 * (world - 1) / world / 1e9
                                        / (stage_ms["exchange"] / 1e3), 1),
            "exchange_bytes_per_rank": len(mine) * plan.rows * plan.cols * 8 * (world - 1) // world}
           if "exchange" in stage_ms else {}),
        "e2e": {"value": round(2 * plan.M * plan.rows * plan.cols * plan.K / 1e9 / (e2e_ms / 1e3), 3),
                "unit": "Gop/s", "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        # per rank and step: prep_B, entangle + GEMM per owned stream, diag reset + check, recover
        "gpu_launches": (1 + 2 * len(mine) + 2 + 1) * args.steps,  # (+ the symmetric-memory barrier when fused)
        "clocks": clk.summary(),
        "correctness": {"flagged_positions": flagged, "recovery_checksum_equal": ok},
    }
    if fs is not None:
        line["failstop"] = fs
    if world == 1:
        ovh = c5_overhead(be, plan, inp, stage_ms)
        line["overhead"] = ovh
        line["overhead_pct"] = ovh["pct"]
    import oracle as O

    n = ORACLE_SAMPLE["c5"][0]
    keep = {}
    O.set_threads(1)
    dt, work, what = c5_oracle_sample(plan, n, keep)
    if world == 1:
        nt = O.max_threads()
        O.set_threads(nt)
        dt2, work2, _ = c5_oracle_sample(plan, n)
        O.set_threads(1)
        line["cpu_baseline"] = {"value": round(work / dt, 6), "unit": "Gop/s", "cores": 1, "kind": "oracle",
                                "sample": what, "seconds": round(dt, 3), "cpu": _cpu_model(),
                                "all_cores": {"value": round(work2 / dt2, 6), "cores": nt, "seconds": round(dt2, 3),
                                              "how": "the oracle's GEMM outer loop split over nproc threads"}}
    # rank 0's checked slice starts at position 0: row 0 of every stream, first n columns
    lo, dchk = res["check_slice"]
    line["correctness"]["oracle_rows_equal"] = bool(
        lo == 0 and all(t.numel() >= n for t in dchk)
        and (np.stack([t[:n].cpu().numpy() for t in dchk]) == keep["d"]).all())
    line["correctness"]["oracle_sample"] = what
    return line


def graph_stage_ms(W, nrot, reps, flush_l2):
    """Median device time of every stage inside the replayed step graph.  For
    stage j the step is captured with exactly two external event-record nodes,
    right before and right after stage j (all other stages present, none
    bracketed), so each stage's number carries one event pair's overhead
    instead of every stage boundary's (round 1 bracketed all stages in one
    capture: ~7 us of node overhead per stage, the stage times summed to more
    than the step)."""
    import torch

    names = [nm for nm, _ in W.stages(0)]
    times = {nm: [] for nm in names}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush_l2 else None
    for j, nm in enumerate(names):
        for i in range(nrot):
            e0 = torch.cuda.Event(enable_timing=True, external=True)
            e1 = torch.cuda.Event(enable_timing=True, external=True)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for jj, (_, f) in enumerate(W.stages(i)):
                    if jj == j:
                        e0.record()
                    f()
                    if jj == j:
                        e1.record()
            g.replay()
            torch.cuda.synchronize()
            for _ in range(reps):
                if flush is not None:
                    flush.fill_(i & 0xff)
                g.replay()
                torch.cuda.synchronize()
                times[nm].append(e0.elapsed_time(e1))
            del g
    return {nm: sorted(v)[len(v) // 2] for nm, v in times.items()}


def event_pair_overhead_ms(W, reps, flush_l2):
    """What an event-record pair adds to a bracketed interval inside the step
    graph: the same capture with an EMPTY pair (nothing between the two
    events) after the first stage; median over replays.  Reported next to
    stages_ms (which are not corrected by it)."""
    import torch

    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush_l2 else None
    e0 = torch.cuda.Event(enable_timing=True, external=True)
    e1 = torch.cuda.Event(enable_timing=True, external=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for jj, (_, f) in enumerate(W.stages(0)):
            f()
            if jj == 0:
                e0.record()
                e1.record()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1)
        g.replay()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del g
    return sorted(ts)[len(ts) // 2]


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1604_04740_b200 as ne

    ne.lib()
    torch.cuda.set_device(local_rank)
    W = make_workload(args, rank, world)
    W.overlap = bool(args.overlap)
    torch.cuda.synchronize()
    # a step with a collective inside (C2 halo, C4 all_gather at N > 1) is
    # timed as eager launches: the collective is not captured into the graph
    use_graph = bool(args.graph) and not (world > 1 and W.has_collective)
    W.eager_only = not use_graph

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up
    for i in range(args.warmup):
        for _, f in W.stages(i):
            f()
    torch.cuda.synchronize()

    # timed region: per-stage CUDA events on the launching (current) stream
    names = [nm for nm, _ in W.stages(0)]
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)] for _ in range(args.steps)]
    clk = ClockSampler(local_rank)
    clk.start()
    barrier()
    torch.cuda.synchronize()
    t_host0 = time.perf_counter()
    for i in range(args.steps):
        st = W.stages(i)
        ev[i][0].record()
        for j, (_, f) in enumerate(st):
            f()
            ev[i][j + 1].record()
    torch.cuda.synchronize()
    barrier()
    t_host1 = time.perf_counter()

    total_ms = sum(ev[i][0].elapsed_time(ev[i][-1]) for i in range(args.steps))
    stage_ms = {nm: sum(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(args.steps)) / args.steps
                for j, nm in enumerate(names)}
    eager_ms = total_ms / args.steps
    flush_l2 = W.e2e_bytes() < (512 << 20)
    if use_graph:
        # the same steps captured once per recovered stream r and replayed: removes
        # the per-call host launch overhead of launch-bound configs (C1, C2)
        graphs = []
        nrot = getattr(W, "M", 1)
        for i in range(nrot):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                W.run_step(i)
            graphs.append(g)
        for i in range(args.warmup):
            graphs[i % nrot].replay()
        torch.cuda.synchronize()
        barrier()
        clk.stop()   # the clock record covers the timed graph replays (the reported number)
        clk = ClockSampler(local_rank)
        clk.start()
        if flush_l2:
            # working set smaller than L2: every timed step starts cold — a 512 MB
            # write evicts the previous step's data, outside the step's own events
            flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for i in range(args.steps):
                flush.fill_(i & 0xff)
                evs[i][0].record()
                graphs[i % nrot].replay()
                evs[i][1].record()
            torch.cuda.synchronize()
            barrier()
            total_ms = sum(a.elapsed_time(b) for a, b in evs)
            del flush
        else:
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            for i in range(args.steps):
                graphs[i % nrot].replay()
            g1.record()
            torch.cuda.synchronize()
            barrier()
            total_ms = g0.elapsed_time(g1)
    clk.stop()
    eager_stage_ms = stage_ms
    if use_graph:
        # per-stage device time inside the replayed step: the same per-r graphs
        # captured again with event-record nodes between the stages (separate
        # graphs, so the timed replays above carry no extra nodes); each replay
        # is synchronised and read, L2 flushed before it when the timed run did
        stage_ms = graph_stage_ms(W, getattr(W, "M", 1), max(3, min(args.steps, 10)), flush_l2)
        ev_overhead = event_pair_overhead_ms(W, max(3, min(args.steps, 10)), flush_l2)
    else:
        ev_overhead = None
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = W.job_work() / (ms_per_step / 1e3)   # the whole job (all ranks) per max-over-ranks step time

    # correctness sentinel of the timed run: no range violation, no flagged position
    dg = ne.diag_read(W.diag)
    # recovered outputs of the last step equal the checked ones
    if getattr(W, "scheme", "entangled") == "abft":
        r_last = (args.steps - 1) % W.M
        rec_ok = bool(torch.equal(W.drec[r_last], W.delta[r_last]))
    else:
        rec_ok = all(bool(torch.equal(a, b)) for a, b in zip(W.drec, W.dout))
    if world > 1:
        # every rank's fault / range counters and recovery verdict (all_reduce of the counters)
        t = torch.tensor([dg["range_violations"], dg["fault_positions"], 0 if rec_ok else 1], device="cuda",
                         dtype=torch.int64)
        dist.all_reduce(t)
        dg = dict(dg, range_violations=int(t[0].item()), fault_positions=int(t[1].item()))
        rec_ok = int(t[2].item()) == 0

    # the oracle on a bounded sample of this rank's inputs (the cpu_baseline
    # leg), and the timed run's outputs (delta and d_hat of the last timed
    # step) compared with it at the sampled positions — before any later
    # measurement reuses the output buffers
    cb = cpu_baseline(args.workload, W)
    oracle_ok = W.oracle_compare()
    if world > 1:
        t = torch.tensor([0 if oracle_ok is False else 1], device="cuda", dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        oracle_ok = None if oracle_ok is None else bool(t.item())

    # end to end through host buffers: pinned H2D inputs, D2H results, every
    # step, pipelined over three CUDA streams (Workload.e2e_pipeline)
    e2e_steps = max(4, min(args.steps, 20))
    W.e2e(2)
    barrier()
    e2e_ms, h2d, d2h = W.e2e(e2e_steps)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    plain = W.plain_times()
    # every rank runs the overhead pipelines (a partitioned step may hold a collective)
    ovh = overhead_block(W, plain) if plain else None
    if world > 1 and ovh is not None:
        t = torch.tensor([ovh["entangled_nofault"]["ms"], ovh["failstop_recover"]["ms"]], device="cuda",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ovh["entangled_nofault"]["ms"], ovh["failstop_recover"]["ms"] = round(float(t[0]), 4), round(float(t[1]), 4)
    if rank != 0:
        return None

    peaks, peak_src = load_peaks()
    info = W.stage_info()
    dom = max((k for k in stage_ms if info.get(k, ("",))[0] in ("hbm", "tensor", "alu")), key=stage_ms.get)
    bound, amount, unit = info[dom]
    achieved = amount / (stage_ms[dom] / 1e3)
    if bound == "hbm":
        peak, runit = peaks["hbm_gbs"], "GB/s"
        peak_note = f"HBM copy bandwidth, {peak_src}"
    elif bound == "tensor":
        peak, runit = peaks["bf16_tflops"] * 2.0, "TOP/s"
        peak_note = f"int8 dense = 2 x bf16 burst ({peaks['bf16_tflops']} TFLOP/s, {peak_src}) x nominal 4.5/2.25"
    else:
        # an exact MAC into a 64-bit accumulator is one IMAD.WIDE (32 x 32 + 64); IMAD.WIDE issues on
        # the fmaheavy pipe at 32 lanes/clk/SM (ncu on the IMAD.WIDE GEMM: fmaheavy 60.4 % busy at
        # 19.0 MAC/clk/SM; the 32-bit IMAD's 64 lanes/clk/SM is quoted in the note)
        peak, runit = 32 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, "TMAC/s"
        peak_note = ("IMAD.WIDE pipe: 32 lanes/clk/SM x 148 SMs x max SM clock (profiles/r02_ncu_summary.md; "
                     "32-bit IMAD: 64 lanes/clk/SM = 2x this)")
    tr = load_traffic().get(f"{W.name}:{dom}")
    traffic = tr["GB"] if tr else None
    xr = W.extra_roofline(dom, stage_ms[dom], peaks) if hasattr(W, "extra_roofline") else None
    srf = step_roofline(W, list(stage_ms), info, peaks, ms_per_step)
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": W.metric_unit,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "strong" if W.partitioned else "weak",
        "vs_baseline": None,
        "dtype": "int32" if getattr(W, "w", 64) == 32 else "int64",  # the containers' arithmetic (w bits)
        "data": "synthetic (counter-based splitmix64 generator, gen/ne_gen.h; no dataset)",
        "config": dict(W.config(), partition=W.partition_note if world > 1 else None,
                       **({"l2": "working set < L2: a 512 MB write flushes L2 before every timed "
                                                   "step, outside that step's CUDA events (per-step timing)"}
                                             if flush_l2 and use_graph else {})),
        "roofline": {"bound": bound, "kernel": dom, "achieved": round(achieved, 2), "peak": round(peak, 1),
                     "unit": runit, "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_unit": "GB per launch, ncu dram__bytes_read.sum + dram__bytes_write.sum "
                                     "(profiles/traffic.json)" if tr else None,
                     "algorithmic_per_launch": f"{amount:.4g} {unit}", "peak_source": peak_note,
                     **({"random_access_floor": xr} if xr else {})},
        "step_roofline": srf,
        "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "stages_timing": ("device time of each stage inside the replayed step graph (one event-record pair around "
                          "that stage per capture, median)"
                          if use_graph else "eager launches, CUDA events between stages"),
        "eager_stages_ms": {k: round(v, 4) for k, v in eager_stage_ms.items()},
        "stages_event_pair_ms": None if ev_overhead is None else round(ev_overhead, 4),
        "launch": ("CUDA graph replay (one graph per recovered stream r)" if use_graph else
                   ("eager (the step contains a collective)" if args.graph else "eager")) +
                  ("; side by side on a second stream: " + ", ".join(
                      f"{s} with {'/'.join(m) if isinstance(m, tuple) else m}" for s, m in W.concurrent.items())
                   if W.overlap and W.concurrent else ""),
        "eager_ms_per_step": round(eager_ms, 4),
        "e2e": {"value": round(W.job_work() / (e2e_ms / 1e3), 3), "unit": W.metric_unit,
                "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "pipelined": "H2D / compute / D2H on three streams, two buffer slots" if W.E2E_PIPELINE
                else "no (one stream; the step is smaller than the enqueue cost of a pipeline)",
                # what the copies alone ask of the host link per step (PCIe; H2D and D2H run concurrently
                # when pipelined): the e2e number is link-bound when these approach the link's rate
                "link_GBs": {"h2d": round(h2d / 1e9 / (e2e_ms / 1e3), 2), "d2h": round(d2h / 1e9 / (e2e_ms / 1e3), 2)}},
        "gpu_launches": W.launches_per_step * args.steps,
        "clocks": clk.summary(),
        "correctness": {"range_violations": dg["range_violations"], "flagged_positions": dg["fault_positions"],
                        "recover_equals_check": rec_ok},
    }
    if ovh is not None:
        line["overhead"] = ovh
        line["overhead_pct"] = ovh["pct"]
    line["timed_host_s"] = round(t_host1 - t_host0, 4)
    if world == 1:
        line["cpu_baseline"] = cb
    line["correctness"]["oracle_rows_equal"] = oracle_ok   # every rank's sample (min over ranks)
    line["correctness"]["oracle_sample"] = cb["sample"] + ("" if world == 1 else " (per rank)")
    return line


def overhead_block(W, plain, reps=10):
    """% overhead vs plain (BASELINE metric; the paper's comparison, F5,
    P:1118-1130) with the scopes stated: the no-fault entangled pipeline (every
    stage but recovery) against each plain pipeline, and the fail-stop
    recovery as its own cost.  Every pipeline is one CUDA graph replayed
    `reps` times (Workload._time), the same launch path on both sides."""
    st = W.stages(0)
    names = [n for n, _ in st if n != "recover"]
    nf = plain.pop("entangled_nofault", None) or (
        W._time(lambda: [f() for n, f in st if n != "recover"], reps), "+".join(names))
    rec = plain.pop("failstop_recover", None) or (W._time(dict(st)["recover"], reps), "recover(one stream lost)")
    pct = {}
    for k, (ms, _) in plain.items():
        if ms and not k.startswith("context") and not k.endswith("_gemm_only"):
            pct[f"nofault_vs_{k}"] = round((nf[0] / ms - 1) * 100, 2)
    pct["failstop_recover_vs_nofault"] = round(rec[0] / nf[0] * 100, 2)
    return {"entangled_nofault": {"ms": round(nf[0], 4), "scope": nf[1]},
            "failstop_recover": {"ms": round(rec[0], 4), "scope": rec[1]},
            "plain": {k: {"ms": None if ms is None else round(ms, 4), "scope": sc} for k, (ms, sc) in plain.items()},
            "pct": pct,
            "timing": f"each pipeline one CUDA graph, {reps} back-to-back replays (CUDA events)"}


def cpu_baseline(workload, W):
    """The oracle as it stands, on one host core, on a bounded sample of the
    workload; for the GEMM configs also with its GEMM's outer loop split over
    every host core, the thread count stated."""
    import oracle as O

    n, _ = ORACLE_SAMPLE[workload]
    O.set_threads(1)
    dt, work, what = W.oracle_sample(n)
    out = {"value": round(work / dt, 6), "unit": W.metric_unit, "cores": 1, "kind": "oracle",
           "sample": what, "seconds": round(dt, 3), "cpu": _cpu_model()}
    if workload in ("c3", "c3p"):
        nt = O.max_threads()
        O.set_threads(nt)
        saved = getattr(W, "_oref", None)
        dt2, work2, _ = W.oracle_sample(n)
        W._oref = saved
        O.set_threads(1)
        out["all_cores"] = {"value": round(work2 / dt2, 6), "cores": nt, "seconds": round(dt2, 3),
                            "how": "the oracle's GEMM outer loop split over nproc threads (same results)"}
    return out


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class _HostOnly:
    """Workload shell for the oracle arm: same config, no device buffers."""


def run_reference(args):
    """The CPU oracle as it stands (plain C, 1 core), each step a bounded sample."""
    cls = WORKLOADS[args.workload] or C3Gemm
    W = cls.__new__(cls)
    # the attributes oracle_sample / work_per_step / config need, without CUDA
    if args.workload in ("c3", "c3p"):
        W.M, W.rows, W.cols, W.K, W.seed, W.algo, W.L, W.limb_bits, W.scheme = \
            3, 4096, 4096, 4096, 2, "tc", 2, 22, "entangled"
        W.true_shape, W.fuse, W.r0, W.rows_global = None, False, 0, 4096
        W.abound, W.bbound, W.wide, W.LB = args.abound, args.bbound, False, 1
        if args.workload == "c3p":
            W.M, W.true_shape = args.streams, (2000, 1200, args.kdim)
            W.rows, W.cols, W.K = 2048, 1280, -(-args.kdim // 128) * 128
            W.limb_bits = {3: 22, 4: 16, 8: 8}.get(W.M, 8)

        class _Cfg:
            l, k = 22, 20
        W.cfg = _Cfg
    elif args.workload == "c4":
        W.M, W.n, W.B, W.seed, W.layout, W.w, W.b0 = 4, 1 << 28, 1024, 3, args.layout, args.w, 0
        W.algo = args.c4algo if (args.layout == "aos" and args.w == 64) else "gather"
        W.vr = (1 << 12) if args.w == 64 else 64

        class _Cfg:
            l, k = (16, 16) if args.w == 64 else (8, 8)
        W.cfg = _Cfg
    elif args.workload == "c5":
        from paper_1604_04740_b200.dist import C5Plan

        plan = C5Plan()
        per_step = ORACLE_SAMPLE["c5"][1]
        for _ in range(args.warmup):
            c5_oracle_sample(plan, per_step)
        tot = work = 0.0
        for _ in range(args.steps):
            dt, wk, what = c5_oracle_sample(plan, per_step)
            tot, work = tot + dt, work + wk
        value = work / tot
        return {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gop/s", "n_gpus": 1,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
                "data": "synthetic (same seeded generator)", "config": {"workload": "C5 (BASELINE configs[4])"},
                "cpu_baseline": {"value": round(value, 6), "unit": "Gop/s", "cores": 1, "kind": "oracle",
                                 "sample": what + " per step", "cpu": _cpu_model()},
                "e2e": {"value": round(value, 6), "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    elif args.workload in ("c2", "c2p"):
        paper = args.workload == "c2p"
        W.M, W.n, W.T, W.seed = (args.streams, 10 ** 6, args.taps, 1) if paper else (3, 65536, 64, 1)
        W.n_global, W.lo, W.halo = W.n, 0, 0
        W.algo, W.paper, W.name = args.conv or ("tc" if paper else "direct"), paper, "C2P" if paper else "C2"
        W.fuse = W.algo == "direct" and bool(args.fuse if args.fuse is not None else 1)
        W.scheme = args.scheme if W.algo == "tc" else "entangled"
        W.L, W.limb_bits = 2, {3: 22, 4: 16, 8: 8}.get(W.M, 8)
        W.block = 256 if W.T >= 256 else 128
        W.kpad = (W.T + W.block - 1 + 127) // 128 * 128

        class _Cfg:
            l, k = {3: (22, 20), 4: (16, 16), 8: (8, 8)}.get(W.M, (8, 8))
        W.cfg = _Cfg
    else:
        W.M, W.n, W.seed, W.w = 3, args.n or 4096, 0, args.w
        W.n_global, W.lo = W.n, 0
        W.fuse = bool(args.fuse if args.fuse is not None else 1)

        class _Cfg:
            l, k = (22, 20) if args.w == 64 else (11, 10)
        W.cfg = _Cfg
    per_step = ORACLE_SAMPLE[args.workload][1]
    for _ in range(args.warmup):
        W.oracle_sample(per_step)
    tot, work, what = 0.0, 0.0, ""
    for _ in range(args.steps):
        dt, wk, what = W.oracle_sample(per_step)
        tot += dt
        work += wk
    value = work / tot
    cfg = W.config()
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": W.metric_unit,
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (same seeded generator)", "config": cfg,
            "cpu_baseline": {"value": round(value, 6), "unit": W.metric_unit, "cores": 1, "kind": "oracle",
                             "sample": what + " per step", "cpu": _cpu_model()},
            "e2e": {"value": round(value, 6), "unit": W.metric_unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    return line


# the other BASELINE configs, measured in the same default run (compact lines
# under "configs"): C1 at its stated N and the HBM-bound 2^27 sweep, C2, C4,
# C5 (one GPU: all 8 streams local; N GPUs: one stream per rank)
CONFIG_SET = (
    ("C1", dict(workload="c1", steps=50)),
    ("C1_n2e27", dict(workload="c1", n=1 << 27, steps=10)),
    ("C2", dict(workload="c2", steps=50)),
    ("C4", dict(workload="c4", steps=5)),
    ("C5", dict(workload="c5", steps=5)),
)
_SUB_DEFAULTS = dict(algo="tc", limbs="plan", scheme="entangled", fuse=None, conv=None, taps=4500, streams=8,
                     kdim=2000, w=64, layout="aos", c4algo="bucket", n=None, failstop="simulated", exchange="auto", graph=1,
                     scaling="strong", abound=64, bbound=64)


def compact(line):
    """The fields of a sub-config line that the configs block keeps."""
    keep = ("value", "unit", "ms_per_step", "steps", "scaling", "dtype", "stages_ms", "gpu_launches",
            "overhead_pct", "correctness")
    out = {k: line[k] for k in keep if k in line}
    out["workload"] = line["config"]["workload"]
    if "roofline" in line:
        out["roofline"] = {k: line["roofline"].get(k) for k in ("bound", "kernel", "achieved", "peak", "unit", "frac",
                                                                  "traffic", "random_access_floor")
                           if k in line["roofline"]}
    if "e2e" in line:
        out["e2e"] = {k: line["e2e"].get(k) for k in ("value", "unit", "ms_per_step", "h2d_bytes_per_step",
                                                      "d2h_bytes_per_step")}
    if "cpu_baseline" in line:
        cb = line["cpu_baseline"]
        out["cpu_baseline"] = {k: cb.get(k) for k in ("value", "unit", "cores", "sample", "all_cores") if k in cb}
    if "clocks" in line:
        out["clocks"] = line["clocks"]
    return out


def step_roofline(W, names, info, peaks, ms_per_step):
    """The whole step against the sum of its stages' own rooflines: each stage's
    algorithmic amount (W.stage_info) at its bound's peak; stages the timed step
    runs side by side (W.concurrent) share the HBM when both are HBM-bound (their
    bytes add) and otherwise overlap (the longer counts).  frac = floor / step."""
    rate = {"hbm": peaks["hbm_gbs"], "tensor": peaks["bf16_tflops"] * 2.0,
            "alu": 32 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12}
    par = W.concurrent if W.overlap else {}
    side_of = {}
    for side, mains in par.items():
        main = next((m for m in (mains if isinstance(mains, tuple) else (mains,)) if m in names), None)
        if side in names and main is not None:
            side_of[main] = side
    sides = set(side_of.values())
    floor, per, missing = 0.0, {}, []
    for nm in names:
        if nm in sides:
            continue
        group = [nm] + ([side_of[nm]] if nm in side_of else [])
        parts = []
        for g in group:
            if g not in info or info[g][0] not in rate:
                missing.append(g)
                continue
            b, amount, _ = info[g]
            parts.append((b, amount, amount / rate[b] * 1e3))
            per[g] = round(amount / rate[b] * 1e3, 4)
        if not parts:
            continue
        if len(parts) > 1 and all(b == "hbm" for b, _, _ in parts):
            floor += sum(a for _, a, _ in parts) / rate["hbm"] * 1e3
        else:
            floor += max(t for _, _, t in parts)
    return {"floor_ms": round(floor, 4), "frac": round(floor / ms_per_step, 4) if ms_per_step else None,
            "stage_floor_ms": per, "unaccounted": missing,
            "basis": "each stage's algorithmic bytes / ops at its roofline's peak (HBM copy bandwidth, int8 tensor, "
                     "IMAD.WIDE pipe); stages run side by side share the HBM when both are HBM-bound"}



def run_configs(args, rank, world, local_rank):
    import argparse as _ap
    import gc

    import torch

    out = {}
    for name, over in CONFIG_SET:
        sub = _ap.Namespace(**{**vars(args), **_SUB_DEFAULTS, **over})
        sub.warmup = max(3, min(args.warmup, 5))
        t0 = time.perf_counter()
        try:
            ln = run_c5(sub, rank, world, local_rank) if sub.workload == "c5" else run_ours(sub, rank, world, local_rank)
            if ln is not None:
                out[name] = dict(compact(ln), wall_s=round(time.perf_counter() - t0, 1))
        except Exception as e:  # noqa: BLE001 — one config failing must not hide the others; reported
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
        gc.collect()
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--algo", default="tc", choices=["tc", "imad", "imad64"],
                    help="c3 GEMM: tcgen05 int8 digits (default); CUDA-core IMAD.WIDE 32 x 32 -> 64 (imad, C3's "
                         "operand fits int32); CUDA-core 64-bit form for any operand (imad64)")
    ap.add_argument("--limbs", default="plan", choices=["plan", "base256"],
                    help="c3: GEMM operand digits: cheapest exact plan (default) or balanced base 256")
    ap.add_argument("--scheme", default="entangled", choices=["entangled", "abft"],
                    help="c3 / c2p: numerical entanglement (default) or the paper's ABFT comparison method")
    ap.add_argument("--fuse", type=int, default=None,
                    help="disentangle/check fused into the op kernel (1) or a separate pass (0); default: the "
                         "measured-faster choice per workload (c1, c2: fused; c3: separate)")
    ap.add_argument("--conv", default=None, choices=["tc", "direct"],
                    help="c2/c2p: tensor-core Toeplitz conv or the direct IMAD kernel (default: the faster one "
                         "measured: direct for c2's 64 taps, tc for c2p)")
    ap.add_argument("--taps", type=int, default=4500, help="c2p: kernel taps (paper: 100-4500)")
    ap.add_argument("--streams", type=int, default=8, help="c2p / c3p: M (paper: 3 or 8)")
    ap.add_argument("--kdim", type=int, default=2000, help="c3p: N, the inner dimension (paper: 200-2000)")
    ap.add_argument("--abound", type=int, default=64,
                    help="c3: A_m ~ U[-abound, abound) (default 64 = configs[2]); wider ranges run the general digit "
                         "plan (ne_gemm_plan_for)")
    ap.add_argument("--bbound", type=int, default=64, help="c3: B ~ U[-bbound, bbound)")
    ap.add_argument("--w", type=int, default=64, choices=[64, 32], help="c1 / c4: container width (P:528-530)")
    ap.add_argument("--layout", default="aos", choices=["aos", "soa"], help="c4: entangled layout at rest")
    ap.add_argument("--c4algo", default="bucket", choices=["gather", "bucket"],
                    help="c4 (AoS, w = 64): the partitioned scatter-reduce (ne_op_permute_inner_check_bucketed: "
                         "no random DRAM gather; default), or the fused gather kernel")
    ap.add_argument("--n", type=int, default=None, help="c1: stream length (default 4096 = configs[0])")
    ap.add_argument("--failstop", default="simulated", choices=["simulated", "exit"],
                    help="c5 at N = M = 8: after the timed steps, the rank of stream 3 exits its process and the "
                         "survivors re-form the world and recover (dist.c5_step_failstop)")
    ap.add_argument("--failstop-timeout", type=float, default=10.0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--exchange", default="auto", choices=["auto", "fused", "nccl"],
                    help="c5: position-major exchange fused into the GEMM epilogue (symmetric memory) or an NCCL "
                         "all_to_all after it; auto = fused when N > 1")
    ap.add_argument("--graph", type=int, default=1, help="time CUDA-graph replays of the step (default) or eager")
    ap.add_argument("--overlap", type=int, default=1,
                    help="run independent stages of the step side by side on a second stream (C3: prep_b with "
                         "entangle, recover with check); 0 = strictly in order")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: partition the stated problem over the ranks (SURVEY 8(e): C1 position ranges, C2 "
                         "ranges + halo, C3 row ranges, C4 stream placement; default) or run one independent replica "
                         "per rank")
    ap.add_argument("--configs", type=int, default=1,
                    help="default workload (c3) only: also measure C1, C1 at 2^27, C2, C4 and C5 in the same run and "
                         "report them under \"configs\" (0: the C3 line alone)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    if os.environ.get("NE_BENCH_SHARE_GPU") == "1":
        # test hook only: exercise the N > 1 code path (barriers, max-over-ranks
        # timing, rank-0 printing) with every rank on cuda:0 over gloo; the
        # numbers of such a run are not measurements
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if os.environ.get("NE_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_c5(args, rank, world, local_rank) if args.workload == "c5" else run_ours(args, rank, world, local_rank)
    default_run = args.workload == "c3" and all(getattr(args, k) == v for k, v in _SUB_DEFAULTS.items()
                                                  if k not in ("taps", "streams", "kdim"))
    if args.configs and default_run:
        import gc

        import torch

        gc.collect()
        torch.cuda.empty_cache()
        cfgs = run_configs(args, rank, world, local_rank)
        if line is not None:
            line["configs"] = cfgs
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
