"""bench.py's CPU legs (the reference arm's timers) on a tiny workload: the 1-core timer and
the all-host-cores bound (one spawned process per core on a series shard).  No GPU."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from conftest import ORACLE_LIB  # noqa: E402
from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig  # noqa: E402


def _data(n=16):
    api = N.NativeApi(ORACLE_LIB)
    return api.make_synthetic(41, n, 88, 4, 0.05)


def test_time_cpu_one_core():
    vals, cats = _data()
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    r = bench.time_cpu(ORACLE_LIB, prof, TrainConfig(batch_size=64, seed=7), vals, cats, budget_s=0.3)
    assert r["cores"] == 1 and r["value"] > 0 and np.isfinite(r["value"])
    assert "epochs" in r["sample"] or "batches" in r["sample"]


def test_time_cpu_all_cores_bound():
    vals, cats = _data()
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    r = bench.time_cpu_all_cores(ORACLE_LIB, prof, TrainConfig(batch_size=64, seed=7), vals, cats, budget_s=0.3)
    assert 1 <= r["cores"] <= 4  # n // 4 shards at most
    assert r["value"] > 0 and np.isfinite(r["value"])
    assert "not the same training problem" in r["note"]


def test_profile_kernels_passes_the_mode_through():
    """bench.py asks for mode 2 (in-graph spans, PDL on); a bool mapping once turned it into
    mode 1 (eager launches with CUDA events), so the reported kernel times were eager-mode."""
    from paper_1907_03329_b200.trainer import Trainer

    calls = []

    class Lib:
        def esrnn_trainer_profile_kernels(self, h, mode):
            calls.append(mode)
            return 0

    class Api:
        lib = Lib()

    t = Trainer.__new__(Trainer)
    t.api, t._h = Api(), None
    t._chk = lambda rc: None
    for m in (0, 1, 2, True, False):
        t.profile_kernels(m)
    assert calls == [0, 1, 2, 1, 0]
    import pytest
    with pytest.raises(ValueError):
        t.profile_kernels(3)
