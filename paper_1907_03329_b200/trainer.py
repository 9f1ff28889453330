"""Host-side mirror of the reference's hot-path API (reference trainer.hpp / data.hpp /
holt_winters.hpp / network.hpp) over the engine C-ABI.

Same names, argument meaning and error behaviour as the C++ reference, so parity tests
read like the reference's own tests:

    FrequencyProfile.defaults(Frequency.Quarterly)      data.hpp:69-99
    TrainConfig(batch_size=..., seed=...)                trainer.hpp:22-44
    Trainer(series, profile, cfg)                        trainer.hpp:159-200
    .train_epoch() / .validate() / .forecast_at(k)       trainer.hpp:234-305
    .batch_loss(b) / .batch_gradients(b)                 trainer.hpp:308-342
    .benchmark_batched_vs_looped()                       trainer.hpp:351-413
    make_batches / pinball_loss / early_stop_check        trainer.hpp:64-120

All device work runs in the CUDA engine (libesrnn_b200.so); this module only marshals
host buffers and reproduces host-side index logic (window lists, RNG shuffles) where the
reference API exposes it.
"""
from __future__ import annotations

import ctypes as C
import enum
import functools
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from . import errors as E
from .rng import Rng


class Category(enum.IntEnum):  # data.hpp:18
    Demographic = 0
    Finance = 1
    Industry = 2
    Macro = 3
    Micro = 4
    Other = 5


class Frequency(enum.IntEnum):  # data.hpp:19
    Yearly = 0
    Quarterly = 1
    Monthly = 2


@dataclass
class SeriesRecord:  # data.hpp:52-57
    id: str
    values: np.ndarray
    category: Optional[Category] = None
    frequency: Optional[Frequency] = None


@dataclass
class FrequencyProfile:  # data.hpp:60-118
    frequency: Frequency = Frequency.Quarterly
    seasonality_length: int = 4
    horizon: int = 8
    input_window: int = 12
    dilation_blocks: list = field(default_factory=lambda: [[1, 2], [4, 8]])
    hidden_size: int = 40
    min_length: int = 72

    @staticmethod
    def defaults(f: Frequency) -> "FrequencyProfile":
        if f == Frequency.Yearly:
            return FrequencyProfile(f, 1, 6, 6, [[1, 2], [2, 6]], 30, 13)
        if f == Frequency.Quarterly:
            return FrequencyProfile(f, 4, 8, 12, [[1, 2], [4, 8]], 40, 72)
        return FrequencyProfile(f, 12, 18, 24, [[1, 3], [6, 12]], 50, 72)

    def equalized_length(self) -> int:
        return self.min_length + 2 * self.horizon

    def to_c(self) -> N.Profile:
        p = N.Profile()
        p.frequency = int(self.frequency)
        p.seasonality_length = self.seasonality_length
        p.horizon = self.horizon
        p.input_window = self.input_window
        p.hidden_size = self.hidden_size
        p.min_length = self.min_length
        if len(self.dilation_blocks) > N.MAX_BLOCKS:
            raise E.ConfigError("profile: too many dilation blocks")
        p.n_blocks = len(self.dilation_blocks)
        layer = 0
        for b, blk in enumerate(self.dilation_blocks):
            p.block_len[b] = len(blk)
            for d in blk:
                if layer >= N.MAX_LAYERS:
                    raise E.ConfigError("profile: too many layers")
                p.dilations[layer] = int(d)
                layer += 1
        return p


@dataclass
class TrainConfig:  # trainer.hpp:22-44 (+ B200 extensions)
    epochs: int = 15
    batch_size: int = 512
    learning_rate_network: float = 1e-3
    learning_rate_per_series: float = 1e-2
    tau: float = 0.5
    gradient_clip: Optional[float] = 20.0
    seed: int = 0
    attach_es_state: bool = True
    patience: int = 0
    min_delta: float = 0.0
    # B200 extensions
    precision: str = "fp64"          # "fp64" (reference arithmetic, default) | "fp32" (performance, opt-in)
    max_batch_size: int = 0          # 0 -> 2048 reference cap
    device: int = 0
    use_graphs: bool = True
    # opt-in ES-RNN level-variability penalty (Smyl's M4 model; absent from the reference,
    # whose loss is pinball only, trainer.hpp:581): 0 = reference behaviour, bit-identical
    level_variability_penalty: float = 0.0

    def to_c(self) -> N.TrainCfg:
        c = N.TrainCfg()
        c.epochs = self.epochs
        c.batch_size = self.batch_size
        c.learning_rate_network = self.learning_rate_network
        c.learning_rate_per_series = self.learning_rate_per_series
        c.tau = self.tau
        c.has_gradient_clip = 0 if self.gradient_clip is None else 1
        c.gradient_clip = 0.0 if self.gradient_clip is None else float(self.gradient_clip)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.attach_es_state = 1 if self.attach_es_state else 0
        c.patience = self.patience
        c.min_delta = self.min_delta
        c.precision = N.FP64 if self.precision == "fp64" else N.FP32
        c.level_variability_penalty = float(self.level_variability_penalty)
        c.max_batch_size = self.max_batch_size
        c.device = self.device
        c.use_graphs = 0 if self.use_graphs else -1
        return c


@dataclass
class DatasetSplit:  # data.hpp:122-126
    train: np.ndarray
    validation: np.ndarray
    test: np.ndarray


def split_train_val_test(values: np.ndarray, horizon: int) -> DatasetSplit:  # data.hpp:128-140
    n, o = len(values), horizon
    if n < 2 * o + 1:
        raise E.InsufficientLengthError(f"split: need at least {2 * o + 1} values, got {n}")
    return DatasetSplit(values[: n - 2 * o], values[n - 2 * o: n - o], values[n - o:])


@dataclass
class PerSeriesParams:  # holt_winters.hpp:26-43
    alpha_raw: float = 0.0
    gamma_raw: float = 0.0
    init_seasonality_raw: np.ndarray = field(default_factory=lambda: np.zeros(1))

    def season_length(self) -> int:
        return len(self.init_seasonality_raw)


@dataclass
class WindowBatch:  # trainer.hpp:50-61
    series_rows: list
    anchors: list
    ids: list = field(default_factory=list)
    mask: Optional[np.ndarray] = None           # (B, O); None -> ones
    inputs: Optional[np.ndarray] = None         # (B, I+6) filled by the pass
    targets: Optional[np.ndarray] = None        # (B, O)
    anchor_levels: Optional[np.ndarray] = None  # (B,)
    seasonality_slices: Optional[np.ndarray] = None  # (B, O)

    def size(self) -> int:
        return len(self.series_rows)


@dataclass
class ValidationResult:  # trainer.hpp:122-127
    ids: list
    forecasts: np.ndarray
    smape_per_series: np.ndarray
    mean_smape: float


@dataclass
class MeanCount:  # metrics.hpp:75-78
    mean: float = 0.0
    count: int = 0


@dataclass
class ReportAggregates:  # metrics.hpp:82-91
    smape_by_category: dict
    smape_by_frequency: dict
    mase_by_category: dict
    mase_by_frequency: dict
    overall_smape: float
    overall_mase: Optional[float]
    total_series: int
    mase_undefined_count: int


def aggregate(categories, frequency: str, smape, mase) -> ReportAggregates:  # metrics.hpp:106-137
    """Per-category / per-frequency running means in row order (the reference's fold), the
    count-weighted overall means (weighted_mean, metrics.hpp:94-104); NaN MASE = nullopt."""
    if len(smape) == 0:
        raise E.ContractError("aggregate: no rows")
    sc, sf, mc, mf = {}, {}, {}, {}
    undefined = 0

    def fold(m, key, v):
        x = m.setdefault(key, MeanCount())
        x.mean = (x.mean * x.count + v) / (x.count + 1)
        x.count += 1

    for c, s_, m_ in zip(categories, smape, mase):
        cname = Category(c).name if c >= 0 else Category.Other.name
        fold(sc, cname, float(s_))
        fold(sf, frequency, float(s_))
        if np.isnan(m_):
            undefined += 1
        else:
            fold(mc, cname, float(m_))
            fold(mf, frequency, float(m_))

    def wmean(m):
        tot = sum(x.count for x in m.values())
        return sum(x.mean * x.count for x in m.values()) / tot

    return ReportAggregates(sc, sf, mc, mf, wmean(sf), wmean(mf) if mf else None, len(smape), undefined)


@dataclass
class EvaluationResult:  # cmd_evaluate's scored rows (commands.hpp:285-338) for model and seasonal-naive
    ids: list
    forecasts: np.ndarray
    smape: np.ndarray
    mase: np.ndarray            # NaN where metrics.hpp:46 returns nullopt
    naive_smape: np.ndarray
    naive_mase: np.ndarray
    totals: np.ndarray          # global sums over ranks (esrnn_trainer_evaluate)
    model: ReportAggregates = None
    naive: ReportAggregates = None

    @property
    def mean_smape(self) -> float:
        return float(self.totals[0] / self.totals[6])

    @property
    def mean_mase(self) -> float:
        return float(self.totals[1] / self.totals[2]) if self.totals[2] else float("nan")


@dataclass
class TrainState:
    """What the reference's checkpoint v1 leaves out (checkpoint.hpp:37-46) and apply_updates /
    make_batches consume: network Adam moments (for_each_param order, trainer.hpp:625-631),
    the global Adam step (:617), per-series moments and steps (:638-650; rows {alpha, gamma,
    seas[S]}), and the trainer RNG (matrix.hpp:173-213) before the next epoch's shuffle."""
    adam_m: np.ndarray
    adam_v: np.ndarray
    net_step: int
    ps_m: np.ndarray      # (n, 2 + S), rows [row_begin, row_begin + n)
    ps_v: np.ndarray
    ps_steps: np.ndarray  # (n,) int64
    rng: str              # std::mt19937_64 text form
    row_begin: int = 0


@dataclass
class ForecastResult:  # trainer.hpp:129-132
    ids: list
    forecasts: np.ndarray


@dataclass
class BenchmarkReport:  # trainer.hpp:134-140
    batched_s: float = 0.0
    looped_s: float = 0.0
    speedup: float = 0.0
    batch_size: int = 0
    n_series: int = 0


@dataclass
class PerSeriesGrad:  # trainer.hpp:146-150
    alpha_raw: float
    gamma_raw: float
    init_seasonality_raw: np.ndarray


@dataclass
class BatchGradients:  # trainer.hpp:143-152
    loss: float
    network: dict
    per_series: dict
    slot_rows: list = field(default_factory=list)


def pinball_loss(predicted, actual, tau: float, mask) -> float:  # trainer.hpp:64-78
    predicted, actual, mask = (np.asarray(x, dtype=np.float64) for x in (predicted, actual, mask))
    if predicted.shape != actual.shape:
        raise E.ShapeError("pinball_loss: shape mismatch")
    if predicted.shape != mask.shape:
        raise E.ShapeError("pinball_loss mask: shape mismatch")
    if not (0.0 < tau < 1.0):
        raise E.ContractError("pinball_loss: tau must be in (0, 1)")
    acc = 0.0
    count = 0.0
    for p, a, m in zip(predicted.ravel(), actual.ravel(), mask.ravel()):
        if m == 0.0:
            continue
        d = a - p
        acc += tau * d if d >= 0.0 else (tau - 1.0) * d
        count += 1.0
    if count == 0.0:
        raise E.ContractError("pinball_loss: all-zero mask, mean undefined")
    return acc / count


def make_batches(windows, series_ids, batch_size: int, horizon: int, rng: Rng):  # trainer.hpp:82-102
    windows = list(windows)
    if not windows:
        raise E.ContractError("make_batches: no windows")
    if batch_size < 1:
        raise E.ConfigError("make_batches: batch_size must be >= 1")
    rng.shuffle(windows)
    out = []
    for start in range(0, len(windows), batch_size):
        chunk = windows[start:start + batch_size]
        out.append(WindowBatch([w[0] for w in chunk], [w[1] for w in chunk],
                               [series_ids[w[0]] for w in chunk], np.ones((len(chunk), horizon))))
    return out


def early_stop_check(history: Sequence[float], patience: int, min_delta: float = 0.0) -> bool:  # :107-120
    if len(history) == 0:
        raise E.ContractError("early_stop_check: empty history")
    if patience <= 0:
        return False
    best, last_improve = history[0], 0
    for i in range(1, len(history)):
        if best - history[i] > min_delta:
            best, last_improve = history[i], i
    return len(history) - 1 - last_improve >= patience


_LAYOUTS: dict = {}  # (library, profile shape) -> (n_values, [(name, rows, cols, offset)])


@functools.lru_cache(maxsize=8)
def _default_ids(n: int) -> list:
    """Ids of array-constructed datasets ("S0", "S1", ...; the synthetic generator's ids)."""
    return [f"S{i}" for i in range(n)]


class Trainer:
    """esrnn::Trainer (trainer.hpp:157-673) backed by a native engine handle."""

    def __init__(self, series, profile: FrequencyProfile, cfg: TrainConfig, *, api: N.NativeApi | None = None,
                 dist: tuple | None = None):
        """dist: series-sharded data parallelism (esrnn_dist), (rank, world, transport[, flags])
        with transport the NCCL unique id (bytes, one process per GPU) or an in-process
        `Group` (api.group(world)); flags N.DIST_FORCE_COLLECTIVE runs the collective step
        at world 1 too."""
        self.api = api if api is not None else N.product_api()
        self._profile = profile
        self._cfg = cfg
        if hasattr(series, "values") and hasattr(series, "categories") and hasattr(series, "ids"):
            # an ingested Dataset (ingest.py): its pinned block goes up without staging
            values, cats = series.values, np.ascontiguousarray(series.categories, dtype=np.int32)
            self._ids_list = list(series.ids)
            self._dataset = series  # keeps the pinned block alive
        elif isinstance(series, tuple):
            values, cats = series
            values = np.ascontiguousarray(values, dtype=np.float64)
            cats = np.ascontiguousarray(cats, dtype=np.int32)
            self._ids_list = None  # "S{i}" ids, built on first use (_ids)
        else:
            series = list(series)
            if not series:
                raise E.ContractError("trainer: no series")
            n = len(series[0].values)
            for s in series:
                if len(s.values) != n:
                    raise E.ConfigError(f'trainer: rectangular batching requires equal series lengths; "{s.id}" '
                                        f"has {len(s.values)} values, expected {n}")
            values = np.ascontiguousarray(np.stack([np.asarray(s.values, dtype=np.float64) for s in series]))
            cats = np.array([-1 if s.category is None else int(s.category) for s in series], dtype=np.int32)
            self._ids_list = [s.id for s in series]
        self._values = values
        self._cats = cats
        c_dist = None
        if dist is not None:
            c_dist = N.Dist()
            c_dist.rank, c_dist.world_size = dist[0], dist[1]
            if isinstance(dist[2], N.Group):
                c_dist.group = dist[2].handle
                self._group = dist[2]  # the group outlives its trainers
            else:
                C.memmove(c_dist.nccl_unique_id, dist[2], 128)
            c_dist.flags = dist[3] if len(dist) > 3 else 0
        h = C.c_void_p()
        p_c, cfg_c = profile.to_c(), cfg.to_c()
        self.api.check(self.api.lib.esrnn_trainer_create(
            C.byref(p_c), C.byref(cfg_c), values.shape[0], values.shape[1], N.dptr(values), N.iptr(cats),
            C.byref(c_dist) if c_dist is not None else None, C.byref(h)))
        self._h = h
        b, e = C.c_int64(), C.c_int64()
        self._chk(self.api.lib.esrnn_trainer_shard(h, C.byref(b), C.byref(e)))
        self.row_begin, self.row_end = b.value, e.value
        # StackWeights layout (network.hpp:62-74) depends only on the profile: asked once per
        # library and profile
        key = (id(self.api), p_c.input_window, p_c.hidden_size, p_c.horizon,
               tuple(p_c.block_len[:p_c.n_blocks]))
        cached = _LAYOUTS.get(key)
        if cached is None:
            na, nv = C.c_int32(), C.c_int64()
            self._chk(self.api.lib.esrnn_trainer_param_count(h, C.byref(na), C.byref(nv)))
            layout = []
            for i in range(na.value):
                info = N.ParamInfo()
                self._chk(self.api.lib.esrnn_trainer_param_info(h, i, C.byref(info)))
                layout.append((info.name.decode(), info.rows, info.cols, info.offset))
            cached = _LAYOUTS[key] = (nv.value, layout)
        self.n_values, self.param_layout = cached[0], list(cached[1])

    # -- plumbing -------------------------------------------------------------------
    @property
    def _ids(self) -> list:
        if self._ids_list is None:
            self._ids_list = _default_ids(self._values.shape[0])  # shared, read-only by convention
        return self._ids_list

    def _chk(self, status):
        self.api.check(status, self._h)

    def close(self):
        if getattr(self, "_h", None):
            self.api.lib.esrnn_trainer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- accessors (trainer.hpp:202-211) ------------------------------------------------
    def profile(self) -> FrequencyProfile:
        return self._profile

    def config(self) -> TrainConfig:
        return self._cfg

    def series_count(self) -> int:
        return self._values.shape[0]

    def series(self, i: int) -> SeriesRecord:
        c = int(self._cats[i])
        return SeriesRecord(self._ids[i], self._values[i].copy(), None if c < 0 else Category(c))

    def split(self, i: int) -> DatasetSplit:
        return split_train_val_test(self._values[i], self._profile.horizon)

    def series_ids(self) -> list:
        return list(self._ids)

    def train_length(self) -> int:
        return self._values.shape[1] - 2 * self._profile.horizon

    def all_windows(self) -> list:  # trainer.hpp:214-223
        I, O, T = self._profile.input_window, self._profile.horizon, self.train_length()
        return [(r, a) for r in range(self.series_count()) for a in range(I - 1, T - O)]

    def weights_flat(self) -> np.ndarray:
        w = np.zeros(self.n_values)
        self._chk(self.api.lib.esrnn_trainer_get_weights(self._h, N.dptr(w), self.n_values))
        return w

    def weights(self) -> dict:
        """StackWeights by name (for_each_param order), as copies."""
        flat = self.weights_flat()
        return {n: flat[o:o + r * c].reshape(r, c).copy() for n, r, c, o in self.param_layout}

    def set_weights(self, w) -> None:  # trainer.hpp:415-432
        if isinstance(w, dict):
            flat = np.zeros(self.n_values)
            if set(w) != {n for n, *_ in self.param_layout}:
                raise E.CheckpointError("checkpoint network shapes incompatible with configuration")
            for n, r, c, o in self.param_layout:
                a = np.asarray(w[n], dtype=np.float64)
                if a.shape != (r, c):
                    raise E.CheckpointError("checkpoint network shapes incompatible with configuration")
                flat[o:o + r * c] = a.ravel()
        else:
            flat = np.ascontiguousarray(w, dtype=np.float64)
        self._chk(self.api.lib.esrnn_trainer_set_weights(self._h, N.dptr(flat), flat.size))

    def per_series_arrays(self):
        n = self.row_end - self.row_begin
        S = self._profile.seasonality_length
        a, g, s = np.zeros(n), np.zeros(n), np.zeros((n, S))
        self._chk(self.api.lib.esrnn_trainer_get_per_series(self._h, self.row_begin, n, N.dptr(a), N.dptr(g),
                                                             N.dptr(s)))
        return a, g, s

    def gather_per_series_arrays(self):
        """Collective on a sharded trainer (every rank calls it): every series' per-series
        parameters, gathered from their owners in dataset order."""
        n, S = self.series_count(), self._profile.seasonality_length
        a, g, s = np.zeros(n), np.zeros(n), np.zeros((n, S))
        self._chk(self.api.lib.esrnn_trainer_gather_per_series(self._h, N.dptr(a), N.dptr(g), N.dptr(s)))
        return a, g, s

    def set_per_series_arrays(self, a, g, s, row_begin=None):
        a, g, s = (np.ascontiguousarray(x, dtype=np.float64) for x in (a, g, s))
        rb = self.row_begin if row_begin is None else row_begin
        self._chk(self.api.lib.esrnn_trainer_set_per_series(self._h, rb, a.shape[0], N.dptr(a), N.dptr(g),
                                                             N.dptr(s)))

    def per_series_params(self, i: int) -> PerSeriesParams:
        S = self._profile.seasonality_length
        a, g, s = np.zeros(1), np.zeros(1), np.zeros(S)
        self._chk(self.api.lib.esrnn_trainer_get_per_series(self._h, i, 1, N.dptr(a), N.dptr(g), N.dptr(s)))
        return PerSeriesParams(float(a[0]), float(g[0]), s)

    def set_per_series_params(self, i: int, p: PerSeriesParams) -> None:
        a, g = np.array([p.alpha_raw]), np.array([p.gamma_raw])
        s = np.ascontiguousarray(p.init_seasonality_raw, dtype=np.float64)
        self._chk(self.api.lib.esrnn_trainer_set_per_series(self._h, i, 1, N.dptr(a), N.dptr(g), N.dptr(s)))

    def set_per_series(self, by_id: dict) -> None:  # trainer.hpp:434-445
        S = self._profile.seasonality_length
        for r in range(self.row_begin, self.row_end):
            sid = self._ids[r]
            if sid not in by_id:
                raise E.CheckpointError(f'checkpoint missing per-series parameters for "{sid}"')
            if by_id[sid].season_length() != S:
                raise E.CheckpointError(f'checkpoint season length incompatible for "{sid}"')
        for r in range(self.row_begin, self.row_end):
            self.set_per_series_params(r, by_id[self._ids[r]])

    def hw_state(self, row: int, t_len: int):
        S = self._profile.seasonality_length
        lv, se = np.zeros(t_len), np.zeros(t_len + S)
        self._chk(self.api.lib.esrnn_trainer_hw_state(self._h, row, t_len, N.dptr(lv), N.dptr(se)))
        return lv, se

    # -- hot path ----------------------------------------------------------------------
    def train_epoch(self) -> float:  # trainer.hpp:234-243
        out = C.c_double()
        self._chk(self.api.lib.esrnn_trainer_train_epoch(self._h, C.byref(out)))
        return out.value

    def _run_batch(self, batch: WindowBatch, flags: int, want_grads_out: bool):
        B = batch.size()
        O = self._profile.horizon
        I, S = self._profile.input_window, self._profile.seasonality_length
        rows = np.ascontiguousarray(batch.series_rows, dtype=np.int32)
        anchors = np.ascontiguousarray(batch.anchors, dtype=np.int32)
        mask = None
        if batch.mask is not None:
            mask = np.ascontiguousarray(batch.mask, dtype=np.float64)
            if mask.shape != (B, O):
                raise E.ShapeError(f"batch: mask shape ({mask.shape[0]}, {mask.shape[1] if mask.ndim > 1 else 1})")
        loss, mc = C.c_double(), C.c_double()
        inputs = np.zeros((B, I + N.NUM_CATEGORIES))
        targets = np.zeros((B, O))
        seas = np.zeros((B, O))
        levels = np.zeros(B)
        gnet = np.zeros(self.n_values) if want_grads_out else None
        nslots = C.c_int32()
        slot_rows = np.zeros(max(B, 1), dtype=np.int32)
        gps = np.zeros((max(B, 1), 2 + S)) if want_grads_out else None
        self._chk(self.api.lib.esrnn_trainer_run_batch(
            self._h, B, N.iptr(rows), N.iptr(anchors), N.dptr(mask), flags, C.byref(loss), C.byref(mc),
            N.dptr(inputs), N.dptr(targets), N.dptr(seas), N.dptr(levels), N.dptr(gnet), C.byref(nslots),
            N.iptr(slot_rows), N.dptr(gps)))
        batch.inputs, batch.targets, batch.seasonality_slices, batch.anchor_levels = inputs, targets, seas, levels
        k = nslots.value
        return loss.value, mc.value, gnet, slot_rows[:k].copy(), (gps[:k].copy() if gps is not None else None)

    def batch_loss(self, batch: WindowBatch) -> float:  # trainer.hpp:338-342
        return self._run_batch(batch, 0, False)[0]

    def batch_gradients(self, batch: WindowBatch) -> BatchGradients:  # trainer.hpp:308-335
        loss, _, gnet, slot_rows, gps = self._run_batch(batch, N.BATCH_GRADS, True)
        net = {n: gnet[o:o + r * c].reshape(r, c).copy() for n, r, c, o in self.param_layout}
        per = {}
        if self._cfg.attach_es_state:
            for s, row in enumerate(slot_rows):
                per[self._ids[row]] = PerSeriesGrad(float(gps[s, 0]), float(gps[s, 1]), gps[s, 2:].copy())
        return BatchGradients(loss, net, per, list(slot_rows))

    def step(self, batch: WindowBatch, update: bool = True):
        """trainer.hpp:593-600 (private in the reference; public here for tests/bench)."""
        loss, mc, *_ = self._run_batch(batch, N.BATCH_GRADS | (N.BATCH_UPDATE if update else 0), False)
        return loss, mc

    def forecast_at(self, drop_tail: int) -> ForecastResult:  # trainer.hpp:248-288
        n = self.row_end - self.row_begin
        out = np.zeros((n, self._profile.horizon))
        self._chk(self.api.lib.esrnn_trainer_forecast(self._h, drop_tail, N.dptr(out)))
        return ForecastResult(self._ids[self.row_begin:self.row_end], out)

    def validate(self) -> ValidationResult:  # trainer.hpp:292-305
        n = self.row_end - self.row_begin
        fc = np.zeros((n, self._profile.horizon))
        sm = np.zeros(n)
        mean = C.c_double()
        self._chk(self.api.lib.esrnn_trainer_validate(self._h, N.dptr(fc), N.dptr(sm), C.byref(mean)))
        return ValidationResult(self._ids[self.row_begin:self.row_end], fc, sm, mean.value)

    def evaluate(self, against_test: bool = True) -> EvaluationResult:
        """cmd_evaluate (commands.hpp:312-338): forecast_at(O) scored against the test block
        (against_test) or forecast_at(2*O) against the validation block, with sMAPE, MASE and
        the seasonal-naive baseline's scores computed on the device."""
        n = self.row_end - self.row_begin
        fc = np.zeros((n, self._profile.horizon))
        arrs = [np.zeros(n) for _ in range(4)]
        tot = np.zeros(8)
        self._chk(self.api.lib.esrnn_trainer_evaluate(self._h, 1 if against_test else 0, N.dptr(fc),
                                                      *[N.dptr(a) for a in arrs], N.dptr(tot)))
        cats = self._cats[self.row_begin:self.row_end]
        fname = self._profile.frequency.name
        res = EvaluationResult(self._ids[self.row_begin:self.row_end], fc, *arrs, tot)
        if n:
            res.model = aggregate(cats, fname, arrs[0], arrs[1])
            res.naive = aggregate(cats, fname, arrs[2], arrs[3])
        return res

    def forward_stack(self, sequence, out_bar=None):
        """network.hpp:190-210 forward_stack over a general input sequence (seq_len, B, I+6) with
        this trainer's StackWeights: the full dilated recurrence.  Returns the (B, O) output, or
        with `out_bar` (B, O) the tuple (out, weights_bar by name, inputs_bar) of the tape's
        reverse-mode adjoints."""
        x = np.ascontiguousarray(sequence, dtype=np.float64)
        if x.ndim != 3 or x.shape[0] < 1:
            raise E.ContractError("forward_stack: empty sequence")
        T, B, width = x.shape
        if width != self._profile.input_window + 6:
            raise E.ShapeError(f"forward_stack: input width {width}, expected {self._profile.input_window + 6}")
        out = np.zeros((B, self._profile.horizon))
        if out_bar is None:
            self._chk(self.api.lib.esrnn_trainer_forward_stack(self._h, T, B, N.dptr(x), N.dptr(out), None, None,
                                                               None))
            return out
        ob = np.ascontiguousarray(out_bar, dtype=np.float64).reshape(B, self._profile.horizon)
        wb = np.zeros(self.n_values)
        xb = np.zeros_like(x)
        self._chk(self.api.lib.esrnn_trainer_forward_stack(self._h, T, B, N.dptr(x), N.dptr(out), N.dptr(ob),
                                                           N.dptr(wb), N.dptr(xb)))
        return out, {n: wb[o:o + r * c].reshape(r, c) for n, r, c, o in self.param_layout}, xb

    def train_state(self) -> TrainState:
        n = self.row_end - self.row_begin
        S = self._profile.seasonality_length
        m, v = np.zeros(self.n_values), np.zeros(self.n_values)
        pm, pv = np.zeros((n, 2 + S)), np.zeros((n, 2 + S))
        steps = np.zeros(n, dtype=np.int64)
        net = C.c_int64()
        buf = C.create_string_buffer(N.RNG_TEXT_MAX)
        lp = C.POINTER(C.c_int64)
        self._chk(self.api.lib.esrnn_trainer_get_train_state(
            self._h, N.dptr(m), N.dptr(v), self.n_values, self.row_begin, n, N.dptr(pm), N.dptr(pv),
            steps.ctypes.data_as(lp), C.byref(net), buf, N.RNG_TEXT_MAX))
        return TrainState(m, v, int(net.value), pm, pv, steps, buf.value.decode(), self.row_begin)

    def set_train_state(self, ts: TrainState) -> None:
        S = self._profile.seasonality_length
        pm = np.ascontiguousarray(ts.ps_m, dtype=np.float64).reshape(-1, 2 + S)
        pv = np.ascontiguousarray(ts.ps_v, dtype=np.float64).reshape(-1, 2 + S)
        steps = np.ascontiguousarray(ts.ps_steps, dtype=np.int64)
        m = np.ascontiguousarray(ts.adam_m, dtype=np.float64)
        v = np.ascontiguousarray(ts.adam_v, dtype=np.float64)
        self._chk(self.api.lib.esrnn_trainer_set_train_state(
            self._h, N.dptr(m), N.dptr(v), m.size, ts.row_begin, pm.shape[0], N.dptr(pm), N.dptr(pv),
            steps.ctypes.data_as(C.POINTER(C.c_int64)), int(ts.net_step), ts.rng.encode()))

    def last_epoch_windows(self) -> list:
        """Global shuffled (row, anchor) order consumed by the last train_epoch."""
        I, O, T = self._profile.input_window, self._profile.horizon, self.train_length()
        n = self.series_count() * (T - O - I + 1)
        r, a = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        self._chk(self.api.lib.esrnn_trainer_last_epoch_windows(self._h, N.iptr(r), N.iptr(a), n))
        return list(zip(r.tolist(), a.tolist()))

    def last_device_ms(self) -> float:
        ms = C.c_double()
        self._chk(self.api.lib.esrnn_trainer_last_device_ms(self._h, C.byref(ms)))
        return ms.value

    def kernel_launches(self) -> int:
        n = C.c_int64()
        self._chk(self.api.lib.esrnn_trainer_kernel_launches(self._h, C.byref(n)))
        return n.value

    KERNEL_CLASSES = ("unused0", "tile", "finish", "unused3", "adam", "finalize", "forecast_scan",
                      "forecast_tile")

    def profile_kernels(self, mode: int) -> None:
        """0: off; 1 (or True): per-kernel CUDA events, eager launches without PDL; 2: in-graph
        global-timer spans of every step's kernels (graph + PDL, the timed configuration)."""
        mode = int(mode)
        if mode not in (0, 1, 2):
            raise ValueError(f"profile_kernels mode must be 0, 1 or 2, got {mode}")
        self._chk(self.api.lib.esrnn_trainer_profile_kernels(self._h, mode))

    def kernel_times(self) -> dict:
        ms = np.zeros(8)
        n = (C.c_int64 * 8)()
        self._chk(self.api.lib.esrnn_trainer_kernel_times(self._h, N.dptr(ms), n))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(self.KERNEL_CLASSES)}

    def benchmark_batched_vs_looped(self) -> BenchmarkReport:  # trainer.hpp:351-413
        windows = self.all_windows()
        O = self._profile.horizon

        def batches_of(bs):
            return [WindowBatch([w[0] for w in windows[s:s + bs]], [w[1] for w in windows[s:s + bs]],
                                ["w"] * len(windows[s:s + bs]), np.ones((len(windows[s:s + bs]), O)))
                    for s in range(0, len(windows), bs)]

        def timed_epoch(batches):
            t0 = time.perf_counter()
            acc = weight = 0.0
            for b in batches:
                loss, mc = self.step(b, update=False)
                acc += loss * mc
                weight += mc
            return acc / weight, time.perf_counter() - t0

        batched, looped = batches_of(self._cfg.batch_size), batches_of(1)
        self.step(batched[0], update=False)
        self.step(looped[0], update=False)
        sb = sl = float("inf")
        lb = ll = 0.0
        for _ in range(3):
            lb, t_b = timed_epoch(batched)
            ll, t_l = timed_epoch(looped)
            sb, sl = min(sb, t_b), min(sl, t_l)
        rel = abs(lb - ll) / max(1e-30, abs(ll))
        if rel > 1e-6:
            raise E.EquivalenceError(f"benchmark: batched loss {lb} vs looped {ll} differ beyond 1e-6; timing withheld")
        return BenchmarkReport(sb, sl, sl / sb, self._cfg.batch_size, self.series_count())
