"""GPU: the C++ host mirror (csrc/host/ensei_b200.hpp) called like REF's own API,
side by side with the compiled reference (tools/cpp_mirror_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "cpp_mirror_check")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/cpp_mirror_check not built")
def test_cpp_mirror_matches_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp mirror ok" in r.stdout
