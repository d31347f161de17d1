import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long CPU-only exhaustive pin (still part of the CPU suite)")


def golden(name):
    """Rows of a tests/golden fixture, comments stripped, '|' separates groups."""
    rows = []
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            rows.append([grp.split() for grp in line.split("|")])
    return rows


@pytest.fixture(scope="session")
def O():
    import oracle

    oracle.lib()
    oracle.set_threads(oracle.max_threads())  # the GEMM's outer loop split over host cores (same results)
    return oracle
