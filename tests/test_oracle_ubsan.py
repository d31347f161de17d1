"""The oracle under UndefinedBehaviorSanitizer: the oracle's pins
and exhaustive checks re-run in a subprocess against liboracle_ubsan.so (the
same C sources built with -fsanitize=undefined -fno-sanitize-recover=all, so
any signed overflow, invalid shift, misaligned or out-of-bounds index the
sanitizer sees aborts the run).  Pass = that pytest run exits 0 with no
"runtime error" report."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists("/usr/bin/gcc"), reason="system gcc (libubsan) not present")
def test_oracle_pins_clean_under_ubsan():
    env = dict(os.environ, NE_ORACLE_UBSAN="1", UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                        "tests/test_oracle_pins.py", "tests/test_oracle_abft.py", "tests/test_oracle_exhaustive.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "runtime error" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    import oracle

    assert oracle.UBSAN is False   # this process still uses the plain build


@pytest.mark.skipif(not os.path.exists("/usr/bin/gcc"), reason="system gcc (libubsan) not present")
def test_ubsan_build_flags_catch_signed_overflow(tmp_path):
    """The sanitizer is live with the flags the oracle build uses: a signed
    overflow aborts with a runtime-error report."""
    src = tmp_path / "ovf.c"
    src.write_text("#include <stdint.h>\nint main(int c, char** v) { int64_t x = INT64_MAX - 1 + c; "
                   "(void)v; return (int)((x + 1) & 1); }\n")
    exe = tmp_path / "ovf"
    subprocess.check_call(["/usr/bin/gcc", "-O1", "-fsanitize=undefined", "-fno-sanitize-recover=all", str(src),
                           "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode != 0 and "runtime error" in r.stderr
