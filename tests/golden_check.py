"""Replay a golden fixture (tests/golden/*.json, produced by the reference) through any
implementation of the C-ABI and compare.  Used by tests/test_oracle.py (plain-C oracle,
CPU) and tests/test_gpu_parity.py (CUDA engine, fp64 and fp32)."""
import json
from pathlib import Path

import numpy as np

from conftest import PROFILES
from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch

GOLDEN = Path(__file__).resolve().parent / "golden"
FIXTURES = ["tiny", "quarterly", "yearly", "monthly"]


def load(name):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def _err(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(b))), 1e-300) if b.size else 1.0
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0


def _cmp_array(got, ref, tol, what):
    got = np.asarray(got, dtype=np.float64).ravel()
    if isinstance(ref, dict):  # summary of a large array
        assert got.size == ref["n"], what
        np.testing.assert_allclose(got[ref["idx"]], ref["val"], rtol=tol, atol=tol * ref["absmax"], err_msg=what)
        assert abs(got.sum() - ref["sum"]) <= tol * max(ref["absmax"] * got.size ** 0.5, 1e-300) + tol * abs(ref["sum"]), what
        assert abs(np.sqrt((got * got).sum()) - ref["l2"]) <= tol * ref["l2"] + 1e-300, what
    else:
        ref = np.asarray(ref, dtype=np.float64).ravel()
        assert got.size == ref.size, (what, got.size, ref.size)
        assert _err(got, ref) <= tol, (what, _err(got, ref))


def check(api, name, precision="fp64", tol=1e-10, tol_train=None, check_windows=True):
    fx = load(name)
    prof = PROFILES[fx["profile"]][0]
    vals = np.array(fx["values"])
    cats = np.array(fx["categories"], dtype=np.int32)
    cfg = TrainConfig(seed=fx["train_seed"], batch_size=fx["batch_size"], precision=precision)
    tr = Trainer((vals, cats), prof, cfg, api=api)
    # init_stack_weights RNG consumption (network.hpp:89-116)
    _cmp_array(tr.weights_flat(), fx["init_weights"], 1e-15 if precision == "fp64" else 1e-7, "init_weights")
    bt = fx["batch"]
    b = WindowBatch(list(bt["rows"]), list(bt["anchors"]), mask=np.array(bt["mask"]))
    g = tr.batch_gradients(b)
    assert abs(g.loss - bt["loss"]) <= tol * abs(bt["loss"]), ("loss", g.loss, bt["loss"])
    for f in ("inputs", "targets", "seasonality_slices", "anchor_levels"):
        _cmp_array(getattr(b, f), bt[f], tol, f)
    assert [int(x) for x in g.slot_rows] == bt["slot_rows"]
    for k, v in bt["net_grads"].items():
        _cmp_array(g.network[k], v, tol * 10, "grad " + k)
    for sid, v in bt["per_series_grads"].items():
        p = g.per_series[sid]
        got = [p.alpha_raw, p.gamma_raw, *p.init_seasonality_raw.tolist()]
        assert _err(got, v) <= tol * 100, ("ps grad", sid, _err(got, v))
    # two training epochs: losses, window order (bit-exact), parameters, validation
    tt = tol_train if tol_train is not None else tol * 100
    for i, ref in enumerate(fx["epoch_losses"]):
        l = tr.train_epoch()
        assert abs(l - ref) <= tt * abs(ref), ("epoch loss", i, l, ref)
    if check_windows:
        order = tr.last_epoch_windows()
        assert len(order) == fx["n_windows"]
        assert [list(x) for x in order[:512]] == fx["last_epoch_windows"]
    _cmp_array(tr.weights_flat(), fx["after_weights"], tt * 10, "after_weights")
    a, gm, sr = tr.per_series_arrays()
    ref_ps = fx["after_per_series"]
    _cmp_array(np.c_[a, gm, sr], np.c_[ref_ps["alpha_raw"], ref_ps["gamma_raw"], ref_ps["seas_raw"]], tt * 10,
               "after_per_series")
    v = tr.validate()
    assert abs(v.mean_smape - fx["validate"]["mean_smape"]) <= tt * 10 * fx["validate"]["mean_smape"]
    _cmp_array(v.forecasts, fx["validate"]["forecasts"], tt * 10, "validate forecasts")
    _cmp_array(tr.forecast_at(0).forecasts, fx["forecast_at_0"], tt * 10, "forecast_at(0)")
    for r, (lv, se) in fx["hw_state_after"].items():
        glv, gse = tr.hw_state(int(r), fx["length"])
        _cmp_array(glv, lv, tt * 10, "hw levels")
        _cmp_array(gse, se, tt * 10, "hw seasonalities")
    return tr
