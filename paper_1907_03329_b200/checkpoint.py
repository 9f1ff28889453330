"""Checkpoints: the reference's JSON model file (checkpoint.hpp:17-143, format
"esrnn-checkpoint" version 1) plus an optional "training_state" object for exact resume.

The reference stores the profile shape, every named network array and the raw per-series
parameters, but neither Adam state nor the trainer RNG (checkpoint.hpp:37-46), so training
cannot resume exactly.  Files written here hold the same v1 fields as
the reference's save_checkpoint, with the same values (doubles round-trip exactly) and the
same key order (nlohmann::json objects are key-sorted, so keys are written sorted); the
reference's load_checkpoint ignores unknown keys, so it still reads them.  Non-finite
parameters are rejected (nlohmann would write them as null, which its own loader refuses).
They add:

    "training_state": {"net_step": int, "rng": "<std::mt19937_64 text>", "epochs": int,
                       "adam": {name: {"m": [...], "v": [...]}},            # for_each_param names
                       "per_series": [{"id", "steps", "m": [a, g, s...], "v": [...]}]}

Host-side file handling, like the reference's; the state itself comes from the device via
Trainer.train_state() (esrnn_trainer_get_train_state).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import errors as E
from .trainer import PerSeriesParams, Trainer, TrainState

CHECKPOINT_VERSION = 1  # checkpoint.hpp:17


@dataclass
class Checkpoint:  # checkpoint.hpp:37-46 (+ training_state)
    frequency: str
    seasonality_length: int
    horizon: int
    input_window: int
    hidden_size: int
    dilation_blocks: list
    network: dict                      # name -> (rows, cols) array
    per_series: list                   # [(id, PerSeriesParams)] in dataset order
    training_state: Optional[dict] = None
    epochs: int = 0


def snapshot(trainer: Trainer, with_training_state: bool = True, epochs: int = 0, gather=None) -> Checkpoint:  # :48-62
    """Checkpoint of `trainer`.  A series-sharded trainer holds only its own rows'
    per-series parameters: they are gathered from their owners by the engine's collective
    (esrnn_trainer_gather_per_series), so EVERY rank must call snapshot.  Its exact-resume
    state additionally needs `gather`, an all-gather of Python objects over the ranks (e.g.
    torch.distributed.all_gather_object wrapped as ``lambda obj: list_of_all_ranks_objs``)."""
    p = trainer.profile()
    sharded = (trainer.row_begin, trainer.row_end) != (0, trainer.series_count())
    ids_all = trainer.series_ids()
    if sharded:
        a, g, s = trainer.gather_per_series_arrays()
    else:
        a, g, s = trainer.per_series_arrays()
    per = [(i, PerSeriesParams(float(a[k]), float(g[k]), s[k].copy())) for k, i in enumerate(ids_all)]
    ck = Checkpoint(p.frequency.name, p.seasonality_length, p.horizon, p.input_window, p.hidden_size,
                    [list(b) for b in p.dilation_blocks], trainer.weights(), per, epochs=epochs)
    if with_training_state:
        if sharded and gather is None:
            raise E.CheckpointError("exact-resume state of a series-sharded trainer needs gather= (the per-series "
                                    "Adam state of other ranks' series lives on those ranks)")
        ts = trainer.train_state()
        ids = ids_all[trainer.row_begin:trainer.row_end]
        ps = [{"id": i, "steps": int(ts.ps_steps[k]), "m": ts.ps_m[k].tolist(), "v": ts.ps_v[k].tolist()}
              for k, i in enumerate(ids)]
        if sharded:
            parts = sorted(gather((trainer.row_begin, ps)), key=lambda x: x[0])
            ps = [e for _, part in parts for e in part]
        adam = {}
        for n, r, c, o in trainer.param_layout:
            adam[n] = {"m": ts.adam_m[o:o + r * c].tolist(), "v": ts.adam_v[o:o + r * c].tolist()}
        ck.training_state = {"net_step": ts.net_step, "rng": ts.rng, "epochs": epochs, "adam": adam,
                             "per_series": ps}
    return ck


def save_checkpoint(path: str, ck: Checkpoint) -> None:  # checkpoint.hpp:64-88
    j = {"format": "esrnn-checkpoint", "version": CHECKPOINT_VERSION, "frequency": ck.frequency,
         "seasonality_length": ck.seasonality_length, "horizon": ck.horizon, "input_window": ck.input_window,
         "hidden_size": ck.hidden_size, "dilation_blocks": ck.dilation_blocks,
         "network": {n: {"rows": int(m.shape[0]), "cols": int(m.shape[1]), "data": np.asarray(m).ravel().tolist()}
                     for n, m in sorted(ck.network.items())},
         "per_series": [{"id": i, "alpha_raw": p.alpha_raw, "gamma_raw": p.gamma_raw,
                         "init_seasonality_raw": list(map(float, p.init_seasonality_raw))} for i, p in ck.per_series]}
    if ck.training_state is not None:
        j["training_state"] = ck.training_state
    try:
        text = json.dumps(j, indent="\t", sort_keys=True, allow_nan=False)  # repr-exact doubles, sorted keys
    except ValueError as e:
        raise E.CheckpointError("checkpoint holds non-finite parameters") from e
    try:
        with open(path, "w") as f:
            f.write(text)
            f.write("\n")
    except OSError as e:
        raise E.Error(f'cannot write checkpoint "{path}"') from e


def load_checkpoint(path: str) -> Checkpoint:  # checkpoint.hpp:90-120
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise E.CheckpointError(f'cannot open checkpoint "{path}"') from e
    except ValueError as e:
        raise E.CheckpointError(f'checkpoint "{path}" is not valid JSON: {e}') from e
    if j.get("format", "") != "esrnn-checkpoint":
        raise E.CheckpointError(f'"{path}" is not an esrnn checkpoint')
    if j.get("version", -1) != CHECKPOINT_VERSION:
        raise E.CheckpointError(f'unsupported checkpoint version in "{path}"')
    try:
        net = {}
        for n, jm in j["network"].items():
            data = np.asarray(jm["data"], dtype=np.float64)
            if data.size != jm["rows"] * jm["cols"]:
                raise E.CheckpointError("matrix data length does not match its shape")
            net[n] = data.reshape(jm["rows"], jm["cols"])
        per = [(js["id"], PerSeriesParams(float(js["alpha_raw"]), float(js["gamma_raw"]),
                                          np.asarray(js["init_seasonality_raw"], dtype=np.float64)))
               for js in j["per_series"]]
        ts = j.get("training_state")
        return Checkpoint(j["frequency"], j["seasonality_length"], j["horizon"], j["input_window"],
                          j["hidden_size"], j["dilation_blocks"], net, per, ts,
                          int(ts.get("epochs", 0)) if ts else 0)
    except KeyError as e:
        raise E.CheckpointError(f'checkpoint "{path}" lacks field {e}') from e


def apply_checkpoint(trainer: Trainer, ck: Checkpoint, resume: bool = True) -> None:  # checkpoint.hpp:123-143
    """Install weights and per-series parameters (the reference's apply_checkpoint); with
    `resume` and a training_state present, also Adam state, steps and the trainer RNG, so
    training continues exactly where the checkpointed run stopped."""
    p = trainer.profile()
    if (ck.frequency != p.frequency.name or ck.seasonality_length != p.seasonality_length
            or ck.horizon != p.horizon or ck.input_window != p.input_window or ck.hidden_size != p.hidden_size
            or [list(b) for b in ck.dilation_blocks] != [list(b) for b in p.dilation_blocks]):
        raise E.CheckpointError("checkpoint profile incompatible with configuration")
    for n, r, c, _ in trainer.param_layout:
        if n not in ck.network:
            raise E.CheckpointError(f'checkpoint missing network array "{n}"')
        if ck.network[n].shape != (r, c):
            raise E.CheckpointError(f'checkpoint array "{n}" has shape {ck.network[n].shape}, expected ({r}, {c})')
    trainer.set_weights({n: ck.network[n] for n, *_ in trainer.param_layout})
    trainer.set_per_series(dict(ck.per_series))
    ts = ck.training_state
    if not resume or ts is None:
        return
    m = np.zeros(trainer.n_values)
    v = np.zeros(trainer.n_values)
    for n, r, c, o in trainer.param_layout:
        a = ts["adam"].get(n)
        if a is None or len(a["m"]) != r * c or len(a["v"]) != r * c:
            raise E.CheckpointError(f'training state missing or misshapen Adam state for "{n}"')
        m[o:o + r * c], v[o:o + r * c] = a["m"], a["v"]
    by_id = {e["id"]: e for e in ts["per_series"]}
    ids = trainer.series_ids()[trainer.row_begin:trainer.row_end]
    S = p.seasonality_length
    pm, pv = np.zeros((len(ids), 2 + S)), np.zeros((len(ids), 2 + S))
    steps = np.zeros(len(ids), dtype=np.int64)
    for k, i in enumerate(ids):
        e = by_id.get(i)
        if e is None:
            raise E.CheckpointError(f'training state has no Adam state for series "{i}"')
        pm[k], pv[k], steps[k] = e["m"], e["v"], e["steps"]
    trainer.set_train_state(TrainState(m, v, int(ts["net_step"]), pm, pv, steps, ts["rng"], trainer.row_begin))


def content_hash(path: str) -> str:  # checkpoint.hpp:146-162
    h = 1469598103934665603
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 14), b""):
            for b in chunk:
                h ^= b
                h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"fnv1a:{h:016x}"
