"""bench.py's side-by-side stages (Workload.run_step): the host logic of the
fork / join, with a stand-in for torch's stream API recording what runs on
which stream — each side stage runs once, on the second stream, forked after
everything before its main stage and joined before the stage after it; with
overlap off (or no matching main stage) the step runs strictly in order."""
import contextlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class _FakeCuda:
    def __init__(self, log):
        self.log, self.cur = log, "main"
        fake = self

        class Stream:
            def __init__(self, name="side"):
                self.name = name

            def wait_event(self, e):
                fake.log.append(("wait", self.name, e.name))

        class Event:
            n = 0

            def __init__(self):
                Event.n += 1
                self.name = f"e{Event.n}"

            def record(self, s):
                fake.log.append(("record", s.name, self.name))

        self.Stream, self.Event, self._main = Stream, Event, Stream("main")

    def current_stream(self):
        return self._main if self.cur == "main" else self.Stream(self.cur)

    @contextlib.contextmanager
    def stream(self, s):
        prev, self.cur = self.cur, s.name
        yield
        self.cur = prev


class _FakeTorch:
    def __init__(self, log):
        self.cuda = _FakeCuda(log)


def _workload(concurrent, names, overlap=True):
    log = []
    W = bench.Workload()
    W.torch = _FakeTorch(log)
    W.concurrent, W.overlap = concurrent, overlap
    W.stages = lambda i: [(nm, (lambda nm=nm: log.append(("run", W.torch.cuda.cur, nm)))) for nm in names]
    return W, log


def _runs(log):
    return [(s, nm) for k, s, nm in log if k == "run"]


def test_c3_pairs_side_by_side():
    W, log = _workload(bench.C3Gemm.concurrent, ["entangle", "prep_b", "gemm", "check", "recover"])
    W.run_step(0)
    assert _runs(log) == [("side", "prep_b"), ("main", "entangle"), ("main", "gemm"), ("side", "recover"),
                          ("main", "check")]
    kinds = [(k, s) for k, s, _ in log]
    # fork (record on main, side waits) before each side stage; join (record on side, main waits) before gemm
    i_fork, i_side = kinds.index(("record", "main")), log.index(("run", "side", "prep_b"))
    assert i_fork < i_side and log[i_fork + 1][:2] == ("wait", "side")
    i_join = next(i for i, x in enumerate(log) if x[:2] == ("record", "side"))
    assert log[i_join + 1][:2] == ("wait", "main") and i_join < log.index(("run", "main", "gemm"))


def test_abft_encode_takes_prep_b_beside_it():
    W, log = _workload(bench.C3Gemm.concurrent, ["encode", "prep_b", "gemm", "check", "recover"])
    W.run_step(0)
    assert ("side", "prep_b") in _runs(log) and ("side", "recover") in _runs(log)


def test_in_order_without_overlap_or_partner():
    names = ["entangle", "prep_b", "gemm", "check", "recover"]
    W, log = _workload(bench.C3Gemm.concurrent, names, overlap=False)
    W.run_step(0)
    assert _runs(log) == [("main", nm) for nm in names] and all(k == "run" for k, _, _ in log)
    W, log = _workload(bench.C2Conv.concurrent, ["entangle", "conv_check", "recover"])
    W.run_step(0)
    assert _runs(log) == [("main", "entangle"), ("main", "conv_check"), ("main", "recover")]


def test_step_roofline_sums_stage_floors():
    """step_roofline: C3's stages at their own peaks, the side-by-side HBM
    pairs (entangle + prep_b, check + recover) sharing the HBM."""
    W = bench.Workload()
    W.concurrent, W.overlap = bench.C3Gemm.concurrent, True
    info = {"entangle": ("hbm", 0.302, "GB"), "prep_b": ("hbm", 0.084, "GB"), "gemm": ("tensor", 0.8246, "TOP"),
            "check": ("hbm", 0.807, "GB"), "recover": ("hbm", 0.671, "GB")}
    peaks = {"hbm_gbs": 6544.0, "bf16_tflops": 1623.3}
    names = ["entangle", "prep_b", "gemm", "check", "recover"]
    r = bench.step_roofline(W, names, info, peaks, 0.565)
    want = (0.302 + 0.084) / 6544 * 1e3 + 0.8246 / 3246.6 * 1e3 + (0.807 + 0.671) / 6544 * 1e3
    assert abs(r["floor_ms"] - want) < 1e-3 and abs(r["frac"] - want / 0.565) < 1e-3 and r["unaccounted"] == []
    W.overlap = False   # in order: the same sum (every pair here is HBM-bound)
    assert abs(bench.step_roofline(W, names, info, peaks, 0.565)["floor_ms"] - want) < 1e-3
    r = bench.step_roofline(W, names + ["halo"], info, peaks, 0.565)
    assert r["unaccounted"] == ["halo"]
