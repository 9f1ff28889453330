"""The reference's trainer-level tests, written against the C++ drop-in header
(include/esrnn_b200/trainer.hpp), run on the B200 engine (tests/cpp/cpp_api_test.cpp)."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_drop_in_api():
    exe = ROOT / "build" / "cpp_api_test"
    assert exe.exists(), "run __graft_entry__.build()"
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed" in r.stdout
