"""GPU: the C++ drop-in (include/nsdc_b200/nsdc_b200.hpp, study.hpp) linked in
one binary with the unmodified reference library: the reference's
integrate_sdc driving the GPU RHS, the device steppers driving the reference
RHS, error behaviour (tests/cpp/shim_parity.cpp); the study harness on the
device path against the reference's study.cpp (tests/cpp/study_parity.cpp).
The binaries are built where /root/reference exists (__graft_entry__.build)
and travel with the repo."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "shim_parity")
STUDY = os.path.join(os.path.dirname(__file__), "cpp", "study_parity")


@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/shim_parity not built")
def test_cpp_dropin_parity(cuda):
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.skipif(not os.path.exists(STUDY), reason="tests/cpp/study_parity not built")
def test_cpp_study_harness_parity(cuda):
    r = subprocess.run([STUDY], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
