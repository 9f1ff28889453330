"""M4 CSV ingestion straight into the engine's upload layout.

    ds = ingest_m4_csv("Monthly-train.csv", "M4-info.csv", FrequencyProfile.defaults(Frequency.Monthly))
    tr = Trainer(ds, profile, cfg)

One native call (esrnn_ingest_m4_csv, paper_1907_03329_b200/csrc/ingest.cpp) does the
reference's cmd_prepare + load_prepared data path -- parse_m4_train_csv, parse_info_csv,
apply_info, frequency filter, length statistics, equalize_lengths
(data.hpp:147-290, commands.hpp:49-175) -- with the train CSV parsed by all host threads
into one pinned block that esrnn_trainer_create uploads without a staging copy.  Values,
ids, categories, statistics and errors (class and message) are the reference's.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E


@dataclass
class LengthStats:  # commands.hpp:77-86
    count: int
    mean: float
    stddev: float
    min: float
    q25: float
    q50: float
    q75: float
    max: float


class Dataset:
    """Equalised series of one frequency: `values` (n x (C + 2O) fp64, a view of the
    engine-owned pinned block), `categories` (int32, data.hpp Category order), `ids`."""

    def __init__(self, api: N.NativeApi, handle, stats: N.IngestStats):
        self.api, self._h = api, handle
        n, length = C.c_int64(), C.c_int32()
        api.check(api.lib.esrnn_dataset_shape(handle, C.byref(n), C.byref(length)))
        self.n, self.length = n.value, length.value
        vp = api.lib.esrnn_dataset_values(handle)
        cp = api.lib.esrnn_dataset_categories(handle)
        self.values = np.ctypeslib.as_array(vp, shape=(self.n, self.length)) if self.n else np.zeros((0, 0))
        self.categories = np.ctypeslib.as_array(cp, shape=(self.n,)) if self.n else np.zeros(0, np.int32)
        self._ids = None
        self.raw_count, self.kept, self.dropped = stats.raw_count, stats.kept, stats.dropped
        self.equalized_length = stats.equalized_length
        self.raw_lengths = LengthStats(stats.raw_count, stats.len_mean, stats.len_stddev, stats.len_min,
                                       stats.len_q25, stats.len_q50, stats.len_q75, stats.len_max)

    @property
    def ids(self) -> list:
        if self._ids is None:
            self._ids = [self.api.lib.esrnn_dataset_id(self._h, i).decode() for i in range(self.n)]
        return self._ids

    def close(self):
        if self._h:
            self.values = self.categories = None
            self.api.lib.esrnn_dataset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def ingest_m4_csv(train_csv: str, info_csv: str, profile, threads: int = 0,
                  api: N.NativeApi | None = None) -> Dataset:
    """cmd_prepare's data path (commands.hpp:141-175) + load_prepared, in one call."""
    api = api if api is not None else N.product_api()
    h = C.c_void_p()
    st = N.IngestStats()
    p = profile.to_c()
    status = api.lib.esrnn_ingest_m4_csv(str(train_csv).encode(), str(info_csv).encode(), int(profile.frequency),
                                         C.byref(p), threads, C.byref(h), C.byref(st))
    if status != 0:
        msg = api.lib.esrnn_ingest_last_error()
        raise N._STATUS.get(status, E.Error)(msg.decode(errors="replace") if msg else f"status {status}")
    return Dataset(api, h, st)
