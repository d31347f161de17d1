"""bench.py's reference arm (--impl reference: the CPU oracle as it stands,
one host core, a bounded sample per step) runs without a GPU for every
workload and prints one JSON line with impl = "reference"; a non-zero rank
(torchrun, N > 1) prints nothing and exits 0."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref(args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", *args], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]


@pytest.mark.parametrize("wl", ["c1", "c2", "c3", "c4", "c5", "c3p", "c2p"])
def test_reference_arm(wl):
    (line,) = _ref(["--workload", wl])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["unit"]


def test_reference_arm_other_ranks_silent():
    assert _ref(["--workload", "c1"], env={"RANK": "1", "WORLD_SIZE": "2"}) == []
