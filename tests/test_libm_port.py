"""The host build of csrc/glibc_math.cuh (the same source the kernels use) against the host
glibc: expf on a dense stride of all 2^32 floats (the full exhaustive sweep is
`tests/native/libm_check.cpp --exhaustive`), exp on random / special ranges incl. the
underflow early-out region."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "libm_check.cpp")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    if not open("/proc/cpuinfo").read().count(" fma "):
        pytest.skip("host libm dispatches the non-FMA exp variant; the port targets __exp_fma")
    exe = str(tmp_path_factory.mktemp("libm") / "libm_check")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_1812_06856_b200", "csrc"),
                    SRC, "-o", exe, "-lm"], check=True)
    return exe


def test_glibc_ports_bit_exact(checker):
    r = subprocess.run([checker], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "exp mismatches: 0" in r.stdout and "expf mismatches: 0" in r.stdout
