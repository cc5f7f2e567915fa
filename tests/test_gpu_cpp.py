"""The drop-in C++ API (include/decmul/*.hpp over libdecmul_gpu.so) running the
reference's own test cases (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_dropin_suite():
    exe = os.path.join(HERE, "cpp", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failures=0" in r.stdout
