"""The C++ drop-in API (include/frpca/frpca.hpp) compiled as reference-style
code (tests/cpp/test_dropin.cpp, built by __graft_entry__.build()) and run on
the B200."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")


def test_cpp_dropin_program(fb):
    if not os.path.exists(EXE):
        from paper_1810_06825_b200 import build
        build.build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
