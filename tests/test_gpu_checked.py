"""The checked build (`make checked`, -DNNVISR_CHECKED -> libnnvisr_checked.so)
stands in for compute-sanitizer, which is closed on the GPU pool: every
shared-memory vector access of the staging kernels must lie in the dynamic
shared memory, every TMA copy must be 16-byte aligned, and in f2t every copy
must land in its stage, read inside a bound frame's planes, and every
converted band and bulk store must stay inside its output buffer; a failed
check traps.  The driver (tools/sanitize_driver.py: TMA and generic paths,
2 segments, padding rows, 5 destinations) must run clean, and a deliberately
short output buffer (NNVISR_F2T_DEBUG=16) must be caught.  The whole GPU
suite under the checked build: tools/checked_tests.sh."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2308_03121_b200", "libnnvisr_checked.so")


def _run(*args, **env):
    e = dict(os.environ, NNVISR_LIBNAME="libnnvisr_checked.so", **env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py"), *args], env=e,
                          capture_output=True, text=True, timeout=300)


@pytest.fixture(scope="module", autouse=True)
def _checked_lib():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", ROOT, "-j4", "checked"])


def test_checked_build_runs_clean():
    r = _run()
    assert r.returncode == 0, r.stdout + r.stderr
    assert "check failed" not in r.stdout + r.stderr
    assert "sanitize driver ok" in r.stdout


def test_checked_build_catches_a_short_output_buffer():
    r = _run("--overflow-control", NNVISR_F2T_DEBUG="16")
    assert r.returncode != 0
    assert "nnvisr check failed" in r.stdout + r.stderr, r.stdout + r.stderr
