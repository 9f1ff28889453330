"""The reference's OWN acceptance suite on the B200 engine.

build/ref_acceptance is /root/reference/proj/tests/acceptance.cpp compiled unmodified, with
the reference's own headers (checkpoint.hpp, commands.hpp, config.hpp, data.hpp,
network.hpp, holt_winters.hpp, metrics.hpp, report.hpp) and exactly one include swapped:
esrnn/trainer.hpp -> the drop-in (tests/cpp/overlay/esrnn/trainer.hpp ->
include/esrnn_b200/trainer.hpp over libesrnn_b200.so).  Built by
paper_1907_03329_b200/build.py (build_reference_acceptance) where the reference tree exists.

Criteria 1-2 exercise the reference's own tape/HW code (no Trainer); 3-9 drive the Trainer
(batched equivalence, batched-vs-looped speedup, overfit, forecast quality, metric goldens,
masking, cmd_train determinism with checkpoint hashes) on the GPU.
"""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_reference_acceptance_suite_on_engine(tmp_path):
    exe = ROOT / "build" / "ref_acceptance"
    assert exe.exists(), "run __graft_entry__.build() where /root/reference exists"
    env = {**os.environ, "TMPDIR": str(tmp_path)}
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900, cwd=tmp_path, env=env)
    print(r.stdout, r.stderr)
    results = dict((int(n), s) for s, n in re.findall(r"\[(PASS|FAIL)\] criterion (\d+)", r.stdout))
    assert sorted(results) == list(range(1, 10)), r.stdout[-3000:]
    assert all(v == "PASS" for v in results.values()), r.stdout[-3000:]
    assert r.returncode == 0
