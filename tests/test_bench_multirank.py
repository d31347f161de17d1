"""bench.py's N > 1 path on one GPU (NE_BENCH_SHARE_GPU=1: every rank on
cuda:0 over gloo — a test hook, its numbers are not measurements): torchrun
with 2 ranks for each BASELINE config, in the default strong-scaling mode
(SURVEY §8(e) partitions: C1 position ranges, C2 ranges + halo exchange, C3
row ranges, C4 stream placement + all_gather, C5 one stream per rank).  Rank
0 prints one JSON line; the line must say strong scaling, no range violation
or flagged position, recovery equal to the check and, for C1-C4, every
rank's outputs equal to the oracle's at its sampled positions."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(args, nproc=2, timeout=600):
    env = dict(os.environ, NE_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(nproc), "--configs", "0", *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("wl,extra", [("c1", []), ("c2", []), ("c3", []), ("c4", ["--steps", "3"])])
def test_bench_two_ranks_partitioned(wl, extra):
    line = _bench(["--workload", wl, "--steps", "5", "--warmup", "3", *extra])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["partition"] and "replicas" not in line["config"]["partition"]
    c = line["correctness"]
    assert c["range_violations"] == 0 and c["flagged_positions"] == 0 and c["recover_equals_check"] is True
    assert c["oracle_rows_equal"] is True
    assert line["value"] > 0 and line["e2e"]["value"] > 0


@pytest.mark.parametrize("wl", ["c2", "c3", "c4"])
def test_bench_four_ranks_partitioned(wl):
    """World 4: C2's halo ring over 4 ranks, C3's 1024-row bands, C4 with one
    stream per rank (the SURVEY §8(e) placement at N = 4)."""
    line = _bench(["--workload", wl, "--steps", "3", "--warmup", "3"], nproc=4, timeout=900)
    assert line["n_gpus"] == 4 and line["scaling"] == "strong"
    c = line["correctness"]
    assert c["range_violations"] == 0 and c["flagged_positions"] == 0 and c["recover_equals_check"] is True
    assert c["oracle_rows_equal"] is True


def test_bench_two_ranks_c5_and_weak_replicas():
    line = _bench(["--workload", "c5", "--steps", "2", "--warmup", "3", "--exchange", "nccl"])
    assert line["n_gpus"] == 2 and line["correctness"]["flagged_positions"] == 0
    assert line["correctness"]["recovery_checksum_equal"] is True
    assert line["correctness"]["oracle_rows_equal"] is True
    line = _bench(["--workload", "c1", "--scaling", "weak", "--steps", "5", "--warmup", "3"])
    assert line["scaling"] == "weak" and line["correctness"]["oracle_rows_equal"] is True
