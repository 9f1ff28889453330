"""Shared fixtures.  Markers: `gpu` (needs a CUDA device and the in-tree engine build).

The oracles under oracle/ are test infrastructure: they are loaded here (and by
bench.py's cpu_baseline leg) as checkers only.
"""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer  # noqa: E402

ORACLE_LIB = ROOT / "oracle" / "liboracle_esrnn.so"
REF_LIB = ROOT / "oracle" / "_ref" / "libesrnn_ref.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the CUDA engine (libesrnn_b200.so)")


def _ensure_oracle():
    if not ORACLE_LIB.exists():
        import subprocess
        subprocess.run(["make", "-s", "liboracle_esrnn.so"], cwd=ROOT / "oracle", check=True)


@pytest.fixture(scope="session")
def oracle():
    _ensure_oracle()
    return N.NativeApi(ORACLE_LIB)


@pytest.fixture(scope="session")
def ref():
    if not REF_LIB.exists():
        pytest.skip("reference shim oracle/_ref/libesrnn_ref.so not built (reference tree absent)")
    return N.NativeApi(REF_LIB)


@pytest.fixture(scope="session")
def engine():
    """The product CUDA engine. Fails loudly (no skip) when the build is missing."""
    return N.product_api()


def tiny_profile():
    # reference tests/test_trainer.cpp:13-22
    return FrequencyProfile(Frequency.Quarterly, 4, 4, 8, [[1, 2]], 6, 20)


PROFILES = {
    "tiny": (tiny_profile(), 28, 4, 0.03),
    "quarterly": (FrequencyProfile.defaults(Frequency.Quarterly), 88, 4, 0.05),
    "yearly": (FrequencyProfile.defaults(Frequency.Yearly), 25, 1, 0.05),
    "monthly": (FrequencyProfile.defaults(Frequency.Monthly), 108, 12, 0.05),
}


def dataset(api, name, n, seed):
    prof, length, s, sigma = PROFILES[name]
    vals, cats = api.make_synthetic(seed, n, length, s, sigma)
    return prof, vals, cats


def make_trainer(api, name, n, data_seed, **cfg):
    prof, vals, cats = dataset(api, name, n, data_seed)
    return Trainer((vals, cats), prof, TrainConfig(**cfg), api=api)


def rel_close(a, b, rtol, atol=0.0):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.all(np.abs(a - b) <= atol + rtol * np.maximum(np.abs(a), np.abs(b)))


def max_rel(a, b, floor=1e-30):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor))) if a.size else 0.0


def tensor_err(a, b):
    """max |a-b| / max(|b|): per-tensor error scaled by the tensor's magnitude."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0
