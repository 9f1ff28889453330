"""The engine's bulk Mersenne twister (csrc/mt64.h) is std::mt19937_64 bit for bit: the
trainer RNG's weight init and epoch shuffles (matrix.hpp:173-213) draw from it."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CSRC = ROOT / "paper_1907_03329_b200" / "csrc"


import pytest


@pytest.mark.parametrize("variant", ["dispatch", "generic"])
def test_mt64_matches_std(tmp_path, variant):
    exe = tmp_path / "mt64_test"
    extra = ["-DESRNN_MT64_GENERIC"] if variant == "generic" else []
    subprocess.run(["g++", "-std=c++17", "-O3", *extra, "-I" + str(CSRC), str(ROOT / "tests" / "cpp" / "mt64_test.cpp"),
                    str(CSRC / "mt64.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mt64: ok" in r.stdout
