"""ctypes binding of the engine C-ABI (include/esrnn_b200.h).

`NativeApi(path)` binds any library implementing the ABI.  The product
(`product_api()`) is the in-tree CUDA build `libesrnn_b200.so`; there is no
fallback — if it is missing, importing the product path raises.  The test
oracles (oracle/liboracle_esrnn.so, oracle/_ref/libesrnn_ref.so) implement the
same ABI and are bound by tests/ only.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import errors as E

MAX_BLOCKS = 8
MAX_LAYERS = 16
NUM_CATEGORIES = 6
FP64, FP32 = 0, 1
BATCH_GRADS, BATCH_UPDATE = 1, 2

PKG_DIR = Path(__file__).resolve().parent
PRODUCT_LIB = PKG_DIR / "libesrnn_b200.so"


class Profile(C.Structure):
    _fields_ = [
        ("frequency", C.c_int32),
        ("seasonality_length", C.c_int32),
        ("horizon", C.c_int32),
        ("input_window", C.c_int32),
        ("hidden_size", C.c_int32),
        ("min_length", C.c_int32),
        ("n_blocks", C.c_int32),
        ("block_len", C.c_int32 * MAX_BLOCKS),
        ("dilations", C.c_int32 * MAX_LAYERS),
    ]


class IngestStats(C.Structure):  # esrnn_ingest_stats
    _fields_ = [("raw_count", C.c_int64), ("kept", C.c_int64), ("dropped", C.c_int64),
                ("equalized_length", C.c_int32), ("len_mean", C.c_double), ("len_stddev", C.c_double),
                ("len_min", C.c_double), ("len_q25", C.c_double), ("len_q50", C.c_double),
                ("len_q75", C.c_double), ("len_max", C.c_double)]


class TrainCfg(C.Structure):
    _fields_ = [
        ("epochs", C.c_int32),
        ("batch_size", C.c_int32),
        ("learning_rate_network", C.c_double),
        ("learning_rate_per_series", C.c_double),
        ("tau", C.c_double),
        ("has_gradient_clip", C.c_int32),
        ("gradient_clip", C.c_double),
        ("seed", C.c_uint64),
        ("attach_es_state", C.c_int32),
        ("patience", C.c_int32),
        ("min_delta", C.c_double),
        ("precision", C.c_int32),
        ("max_batch_size", C.c_int32),
        ("device", C.c_int32),
        ("use_graphs", C.c_int32),
        ("level_variability_penalty", C.c_double),
    ]


class Dist(C.Structure):  # esrnn_dist (ABI 2)
    _fields_ = [("rank", C.c_int32), ("world_size", C.c_int32), ("nccl_unique_id", C.c_uint8 * 128),
                ("flags", C.c_int32), ("group", C.c_void_p)]


DIST_FORCE_COLLECTIVE = 1


class ParamInfo(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("rows", C.c_int32), ("cols", C.c_int32), ("offset", C.c_int64)]


_STATUS = {
    1: E.Error, 2: E.ParseError, 3: E.ValidationError, 4: E.ShapeError,
    5: E.InsufficientLengthError, 6: E.NumericDomainError, 7: E.ConfigError,
    8: E.ContractError, 9: E.EquivalenceError, 10: E.CheckpointError,
    11: E.CudaError, 12: E.NcclError,
}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_vp = C.c_void_p


RNG_TEXT_MAX = 8192  # esrnn_b200.h ESRNN_RNG_TEXT_MAX


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


class NativeApi:
    """One loaded implementation of the ABI."""

    def __init__(self, path: str | os.PathLike):
        path = Path(path)
        if not path.exists():
            raise E.CudaError(f"native library {path} is missing (run __graft_entry__.build())")
        # RTLD_LOCAL: several implementations of the same ABI can coexist in one process
        self.path = path
        self.lib = C.CDLL(str(path), mode=os.RTLD_LOCAL | os.RTLD_NOW)
        L = self.lib
        L.esrnn_version.restype = C.c_char_p
        L.esrnn_abi_version.restype = C.c_int32
        L.esrnn_last_error.restype = C.c_char_p
        L.esrnn_last_error.argtypes = [_vp]
        L.esrnn_trainer_create.argtypes = [C.POINTER(Profile), C.POINTER(TrainCfg), C.c_int64, C.c_int32,
                                           _dp, _ip, C.POINTER(Dist), C.POINTER(_vp)]
        L.esrnn_trainer_destroy.argtypes = [_vp]
        L.esrnn_trainer_destroy.restype = None
        L.esrnn_trainer_shard.argtypes = [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.esrnn_trainer_param_count.argtypes = [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.esrnn_trainer_param_info.argtypes = [_vp, C.c_int32, C.POINTER(ParamInfo)]
        L.esrnn_trainer_get_weights.argtypes = [_vp, _dp, C.c_int64]
        L.esrnn_trainer_set_weights.argtypes = [_vp, _dp, C.c_int64]
        L.esrnn_trainer_get_per_series.argtypes = [_vp, C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.esrnn_trainer_set_per_series.argtypes = [_vp, C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.esrnn_trainer_train_epoch.argtypes = [_vp, _dp]
        L.esrnn_trainer_run_batch.argtypes = [_vp, C.c_int32, _ip, _ip, _dp, C.c_int32, _dp, _dp, _dp, _dp,
                                              _dp, _dp, _dp, _ip, _ip, _dp]
        L.esrnn_trainer_forecast.argtypes = [_vp, C.c_int64, _dp]
        L.esrnn_trainer_validate.argtypes = [_vp, _dp, _dp, _dp]
        L.esrnn_trainer_evaluate.argtypes = [_vp, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp]
        L.esrnn_trainer_forward_stack.argtypes = [_vp, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, _dp]
        _lp = C.POINTER(C.c_int64)
        L.esrnn_trainer_get_train_state.argtypes = [_vp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _lp,
                                                    _lp, C.c_char_p, C.c_int64]
        L.esrnn_trainer_set_train_state.argtypes = [_vp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _lp,
                                                    C.c_int64, C.c_char_p]
        L.esrnn_trainer_hw_state.argtypes = [_vp, C.c_int64, C.c_int64, _dp, _dp]
        L.esrnn_trainer_last_device_ms.argtypes = [_vp, _dp]
        L.esrnn_trainer_last_epoch_windows.argtypes = [_vp, _ip, _ip, C.c_int64]
        L.esrnn_trainer_kernel_launches.argtypes = [_vp, C.POINTER(C.c_int64)]
        L.esrnn_trainer_profile_kernels.argtypes = [_vp, C.c_int32]
        L.esrnn_trainer_kernel_times.argtypes = [_vp, _dp, C.POINTER(C.c_int64)]
        L.esrnn_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        L.esrnn_group_create.argtypes = [C.c_int32, C.POINTER(_vp)]
        L.esrnn_group_destroy.argtypes = [_vp]
        L.esrnn_group_destroy.restype = None
        L.esrnn_trainer_gather_per_series.argtypes = [_vp, _dp, _dp, _dp]
        L.esrnn_release_cached_memory.argtypes = []
        L.esrnn_make_synthetic.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_double, _dp, _ip]
        L.esrnn_ingest_m4_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_int32, C.POINTER(Profile), C.c_int32,
                                          C.POINTER(_vp), C.POINTER(IngestStats)]
        L.esrnn_ingest_m4_csv.restype = C.c_int
        L.esrnn_ingest_last_error.restype = C.c_char_p
        L.esrnn_dataset_shape.argtypes = [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.esrnn_dataset_shape.restype = C.c_int
        L.esrnn_dataset_values.argtypes = [_vp]
        L.esrnn_dataset_values.restype = _dp
        L.esrnn_dataset_categories.argtypes = [_vp]
        L.esrnn_dataset_categories.restype = _ip
        L.esrnn_dataset_id.argtypes = [_vp, C.c_int64]
        L.esrnn_dataset_id.restype = C.c_char_p
        L.esrnn_dataset_destroy.argtypes = [_vp]
        L.esrnn_dataset_destroy.restype = None
        for fn in ("esrnn_trainer_create", "esrnn_trainer_shard", "esrnn_trainer_param_count",
                   "esrnn_trainer_param_info", "esrnn_trainer_get_weights", "esrnn_trainer_set_weights",
                   "esrnn_trainer_get_per_series", "esrnn_trainer_set_per_series", "esrnn_trainer_train_epoch",
                   "esrnn_trainer_run_batch", "esrnn_trainer_forecast", "esrnn_trainer_validate", "esrnn_trainer_evaluate",
                   "esrnn_trainer_get_train_state", "esrnn_trainer_set_train_state", "esrnn_trainer_forward_stack",
                   "esrnn_trainer_hw_state", "esrnn_trainer_last_device_ms", "esrnn_trainer_last_epoch_windows", "esrnn_trainer_kernel_launches",
                   "esrnn_trainer_profile_kernels", "esrnn_trainer_kernel_times", "esrnn_nccl_unique_id", "esrnn_make_synthetic",
                   "esrnn_release_cached_memory", "esrnn_group_create", "esrnn_trainer_gather_per_series"):
            getattr(L, fn).restype = C.c_int

    @property
    def version(self) -> str:
        return self.lib.esrnn_version().decode()

    def check(self, status: int, handle=None) -> None:
        if status == 0:
            return
        msg = self.lib.esrnn_last_error(handle)
        msg = msg.decode(errors="replace") if msg else ""
        raise _STATUS.get(status, E.Error)(msg or f"status {status}")

    def make_synthetic(self, seed: int, n: int, length: int, season_length: int, noise_sigma: float):
        vals = np.zeros((n, length), dtype=np.float64)
        cats = np.zeros(n, dtype=np.int32)
        self.check(self.lib.esrnn_make_synthetic(seed, n, length, season_length, noise_sigma, dptr(vals), iptr(cats)))
        return vals, cats

    def release_cached_memory(self) -> None:
        """Return the engine's cached device / pinned blocks and epoch graphs to CUDA."""
        self.check(self.lib.esrnn_release_cached_memory())

    def group(self, world_size: int) -> "Group":
        """An in-process rank group (esrnn_group_create) for `world_size` sharded trainers."""
        return Group(self, world_size)

    def nccl_unique_id(self) -> bytes:
        buf = (C.c_uint8 * 128)()
        self.check(self.lib.esrnn_nccl_unique_id(buf))
        return bytes(buf)


_PRODUCT: NativeApi | None = None


def product_api() -> NativeApi:
    """The CUDA engine.  Raises if the in-tree build is absent — no CPU fallback."""
    global _PRODUCT
    if _PRODUCT is None:
        _PRODUCT = NativeApi(os.environ.get("ESRNN_B200_LIB", PRODUCT_LIB))
    return _PRODUCT


class Group:
    """esrnn_group: W series-sharded trainers in one process (one host thread each), whose
    per-step collective is the engine's fused in-process reduce kernel instead of NCCL."""

    def __init__(self, api: NativeApi, world_size: int):
        self.api, self.world_size = api, world_size
        h = C.c_void_p()
        api.check(api.lib.esrnn_group_create(world_size, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            self.api.lib.esrnn_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
