"""Opt-in level-variability penalty (B200 extension; BASELINE north_star "pinball loss plus
the level-variability penalty is a fused reduction").  The reference has no such term (its
loss is pinball only, trainer.hpp:581), so there is no reference golden: the oracle's
restatement (oracle/esrnn_oracle.c lvp_series, after Smyl's M4 ES-RNN: the mean squared
second difference of the log levels) is pinned here by
  * weight 0 == the reference (loss and gradients bit-identical to lambda = 0 runs, which
    are themselves pinned to the reference golden vectors),
  * central finite differences of the penalised loss w.r.t. every per-series raw parameter,
  * a closed-form value on a hand-built level path,
  * the reference shim refusing a non-zero weight (the reference cannot compute it).
The engine is checked against this oracle in tests/test_gpu_penalty.py.
"""
import numpy as np
import pytest

from conftest import dataset, tensor_err
from paper_1907_03329_b200 import errors as E
from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch

LAM = 3.0


def _pair(api, name, n, seed, lam, **kw):
    prof, vals, cats = dataset(api, name, n, seed)
    return Trainer((vals, cats), prof, TrainConfig(seed=seed, batch_size=64, level_variability_penalty=lam, **kw),
                   api=api)


def _batch(tr, n=24, seed=0):
    w = tr.all_windows()
    idx = np.random.default_rng(seed).choice(len(w), size=min(n, len(w)), replace=False)
    return [w[i][0] for i in idx], [w[i][1] for i in idx]


def test_zero_weight_is_reference(oracle, ref):
    """lambda = 0 (the default) is the reference: the oracle equals the reference itself."""
    a = _pair(oracle, "quarterly", 8, 3, 0.0)
    prof, vals, cats = dataset(ref, "quarterly", 8, 3)
    b = Trainer((vals, cats), prof, TrainConfig(seed=3, batch_size=64), api=ref)
    rows, anchors = _batch(a)
    ga, gb = a.batch_gradients(WindowBatch(rows, anchors)), b.batch_gradients(WindowBatch(rows, anchors))
    assert abs(ga.loss - gb.loss) <= 1e-13 * abs(gb.loss)
    for k in ga.network:
        assert tensor_err(ga.network[k], gb.network[k]) < 1e-11, k


def _penalty_closed_form(levels, c):
    u = np.log(levels)
    e = u[2:] - 2 * u[1:-1] + u[:-2]
    return c * np.mean(e * e)


@pytest.mark.parametrize("name", ["quarterly", "yearly", "monthly"])
def test_penalty_value_matches_closed_form(oracle, name):
    p0, p1 = _pair(oracle, name, 6, 4, 0.0), _pair(oracle, name, 6, 4, LAM)
    rows, anchors = _batch(p0, 10, 1)
    l0, l1 = p0.batch_loss(WindowBatch(rows, anchors)), p1.batch_loss(WindowBatch(rows, anchors))
    T = p0.train_length()
    M = len(rows) * p0.profile().horizon
    want = 0.0
    for r in sorted(set(rows)):
        lv, _ = p0.hw_state(r, T)
        want += _penalty_closed_form(np.asarray(lv), LAM * p0.profile().horizon * rows.count(r) / M)
    assert abs((l1 - l0) - want) <= 1e-12 * max(1.0, abs(want))


@pytest.mark.parametrize("name", ["quarterly", "yearly"])
def test_penalty_gradient_central_differences(oracle, name):
    """d loss / d raw parameter of the penalised loss vs central differences (the network
    gradient does not depend on the penalty: bit-equal to lambda = 0)."""
    tr, t0 = _pair(oracle, name, 5, 6, LAM), _pair(oracle, name, 5, 6, 0.0)
    rows, anchors = _batch(tr, 12, 2)
    g = tr.batch_gradients(WindowBatch(rows, anchors))
    g0 = t0.batch_gradients(WindowBatch(rows, anchors))
    for k in g.network:
        assert np.array_equal(g.network[k], g0.network[k]), k
    a, gm, s = (x.copy() for x in tr.per_series_arrays())
    ids = tr.series_ids()
    S = s.shape[1]
    worst = 0.0
    for r in sorted(set(rows)):
        ps = g.per_series[ids[r]]
        for which in range(2 + S):
            def loss_at(d):
                aa, gg, ss = a.copy(), gm.copy(), s.copy()
                if which == 0:
                    aa[r] += d
                elif which == 1:
                    gg[r] += d
                else:
                    ss[r, which - 2] += d
                tr.set_per_series_arrays(aa, gg, ss)
                return tr.batch_loss(WindowBatch(rows, anchors))
            h = 1e-6
            fd = (loss_at(h) - loss_at(-h)) / (2 * h)
            an = ps.alpha_raw if which == 0 else ps.gamma_raw if which == 1 else ps.init_seasonality_raw[which - 2]
            worst = max(worst, abs(fd - an) / max(abs(an), 1e-3))
    tr.set_per_series_arrays(a, gm, s)
    assert worst < 1e-5, worst


def test_penalty_changes_per_series_gradients_only_when_attached(oracle):
    tr = _pair(oracle, "quarterly", 6, 5, LAM, attach_es_state=False)
    t0 = _pair(oracle, "quarterly", 6, 5, 0.0, attach_es_state=False)
    rows, anchors = _batch(tr, 12, 3)
    assert tr.batch_loss(WindowBatch(rows, anchors)) == t0.batch_loss(WindowBatch(rows, anchors))


def test_negative_weight_rejected(oracle):
    with pytest.raises(E.ConfigError):
        _pair(oracle, "quarterly", 4, 1, -1.0)


def test_reference_shim_refuses_penalty(ref):
    with pytest.raises(E.ConfigError):
        _pair(ref, "quarterly", 4, 1, LAM)
