"""The host build of the glibc powf / cbrtf ports and of rgb_to_scaled_lab (csrc/glibc_math.cuh,
the same source the GPU conversion kernel uses) against the host glibc: every float operand the
conversion can produce for inputs in [0, 1.5] (4.4e7 powf and 6.2e7 cbrtf operands), random
operands, and 3e6 random colours (tests/native/lab_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "lab_check.cpp")


def test_powf_cbrtf_lab_ports_bit_exact(tmp_path):
    if not open("/proc/cpuinfo").read().count(" fma "):
        pytest.skip("host libm dispatches the non-FMA powf variant; the port targets __powf_fma")
    exe = str(tmp_path / "lab_check")
    # -fno-builtin: keep gcc from folding libm calls with its own (correctly rounded) arithmetic
    subprocess.run(["g++", "-O2", "-fno-builtin", "-ffp-contract=off", "-I",
                    os.path.join(ROOT, "paper_1812_06856_b200", "csrc"), SRC, "-o", exe, "-lm"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "powf operands" in r.stdout and "lab mismatches: 0" in r.stdout
