"""CPU tests pinning the plain-C oracle (oracle/esrnn_oracle.c) to the reference.

1. Golden fixtures generated from the reference itself (tests/golden/make_golden.py).
2. Live diff against the reference compiled from /root/reference (oracle/_ref), when built.
3. The reference's own known-answer tests for this path (test_holt_winters.cpp:36-60,
   test_trainer.cpp:44-51 / acceptance.cpp:453-491, test_trainer.cpp:200-216).
"""
import numpy as np
import pytest

import golden_check
from conftest import PROFILES, dataset, max_rel, tensor_err
from paper_1907_03329_b200 import errors as E
from paper_1907_03329_b200.trainer import (FrequencyProfile, Frequency, TrainConfig, Trainer, WindowBatch,
                                           early_stop_check, make_batches, pinball_loss)
from paper_1907_03329_b200.rng import Rng


@pytest.mark.parametrize("name", golden_check.FIXTURES)
def test_oracle_matches_reference_golden(oracle, name):
    golden_check.check(oracle, name, "fp64", tol=1e-12, tol_train=1e-11)


@pytest.mark.parametrize("name,n,seed", [("tiny", 4, 5), ("quarterly", 6, 9), ("yearly", 30, 2), ("monthly", 4, 3)])
def test_oracle_matches_reference_live(oracle, ref, name, n, seed):
    prof, vals, cats = dataset(ref, name, n, seed)
    cfg = TrainConfig(seed=seed, batch_size=32)
    o, r = (Trainer((vals, cats), prof, cfg, api=a) for a in (oracle, ref))
    assert tensor_err(o.weights_flat(), r.weights_flat()) < 1e-15
    for _ in range(2):
        assert max_rel(o.train_epoch(), r.train_epoch()) < 1e-12
        assert o.last_epoch_windows() == r.last_epoch_windows()
    assert tensor_err(o.weights_flat(), r.weights_flat()) < 1e-11
    assert max_rel(o.validate().mean_smape, r.validate().mean_smape) < 1e-12
    w = o.all_windows()
    b = WindowBatch([x[0] for x in w[:40]], [x[1] for x in w[:40]])
    go, gr = o.batch_gradients(WindowBatch(b.series_rows, b.anchors)), r.batch_gradients(b)
    for k in gr.network:
        assert tensor_err(go.network[k], gr.network[k]) < 1e-11, k


def test_synthetic_generator_matches_reference(oracle, ref):
    """helpers.hpp:148-172 consumed from Rng(41): same categories, values within 1 ulp
    (the reference build contracts to FMA)."""
    for s in (1, 4, 12):
        vo, co = oracle.make_synthetic(41, 20, 40, s, 0.05)
        vr, cr = ref.make_synthetic(41, 20, 40, s, 0.05)
        assert np.array_equal(co, cr)
        assert np.max(np.abs(vo - vr) / np.abs(vr)) < 1e-15


def _single_series_trainer(api, y, S=1, O=1, I=1):
    prof = FrequencyProfile(Frequency.Yearly, S, O, I, [[1]], 2, 1)
    vals = np.array([y + [1.0] * (2 * O + I + O - len(y) + 2)])  # pad so the split holds a window
    return Trainer((vals, np.array([5], dtype=np.int32)), prof, TrainConfig(seed=0), api=api)


def test_hw_two_point_example(oracle):
    """test_holt_winters.cpp:49-60: y=[10,12], S=1, alpha=gamma=0.5 -> levels [10, 11],
    seasonalities [1, 1, 1.1]."""
    tr = _single_series_trainer(oracle, [10.0, 12.0])
    lv, se = tr.hw_state(0, 2)
    np.testing.assert_allclose(lv, [10.0, 11.0], rtol=1e-15)
    np.testing.assert_allclose(se, [1.0, 1.0, 1.1], rtol=1e-15)


def test_hw_alpha_limits(oracle):
    """test_holt_winters.cpp:36-47: alpha -> 1 tracks y; alpha -> 0 carries l0."""
    y = [3.0, 7.0, 2.0, 9.0, 4.0]
    tr = _single_series_trainer(oracle, y)
    tr.set_per_series_arrays([40.0], [-40.0], [[0.0]])
    lv, _ = tr.hw_state(0, 5)
    np.testing.assert_allclose(lv, y, rtol=1e-12)
    tr.set_per_series_arrays([-40.0], [0.0], [[0.0]])
    lv, _ = tr.hw_state(0, 5)
    np.testing.assert_allclose(lv, [3.0] * 5, rtol=1e-12)


def test_hw_rejects_bad_input(oracle):
    """test_holt_winters.cpp:62-67"""
    tr = _single_series_trainer(oracle, [1.0, -2.0])
    with pytest.raises(E.NumericDomainError):
        tr.hw_state(0, 2)


def test_pinball_goldens():
    """test_trainer.cpp:44-51, acceptance.cpp:474-479"""
    one = np.ones((1, 1))
    assert pinball_loss([[2.0]], [[2.0]], 0.5, one) == 0.0
    assert abs(pinball_loss([[0.0]], [[2.0]], 0.5, one) - 1.0) < 1e-15
    assert abs(pinball_loss([[1.0]], [[0.0]], 0.9, one) - 0.1) < 1e-15
    with pytest.raises(E.ContractError):
        pinball_loss([[1.0]], [[0.0]], 0.5, np.zeros((1, 1)))


def test_early_stop_rules():
    """test_trainer.cpp:86-94"""
    assert not early_stop_check([5.0, 4.0, 3.0, 2.0], 2)
    assert early_stop_check([3.0, 3.0, 3.0], 2)
    assert not early_stop_check([3.0, 3.0], 2)
    assert early_stop_check([5.0, 4.875], 1, 0.125)
    assert not early_stop_check([5.0, 4.75], 1, 0.125)
    with pytest.raises(E.ContractError):
        early_stop_check([], 2)


def test_make_batches_partition_and_determinism():
    """test_trainer.cpp:53-84"""
    windows = [(i % 3, 7 + i) for i in range(10)]
    ids = ["a", "b", "c"]
    b1 = make_batches(windows, ids, 4, 4, Rng(5))
    assert [b.size() for b in b1] == [4, 4, 2]
    b2 = make_batches(windows, ids, 4, 4, Rng(5))
    assert all(x.anchors == y.anchors and x.series_rows == y.series_rows for x, y in zip(b1, b2))
    b3 = make_batches(windows, ids, 4, 4, Rng(6))
    assert any(x.anchors != y.anchors for x, y in zip(b1, b3))
    seen = sorted((r, a) for b in b1 for r, a in zip(b.series_rows, b.anchors))
    assert seen == sorted(windows)


def test_python_rng_matches_reference_epoch_order(ref):
    """The Python mirror of Rng/make_batches reproduces the reference's window order:
    the trainer RNG first draws init_stack_weights (network.hpp:89-116), then shuffles."""
    prof, vals, cats = dataset(ref, "tiny", 5, 3)
    tr = Trainer((vals, cats), prof, TrainConfig(seed=42, batch_size=16), api=ref)
    tr.train_epoch()
    rng = Rng(42)
    for _ in range(tr.n_values - sum(r * c for n, r, c, o in tr.param_layout if n.endswith("bias") or n.endswith("nl_b") or n.endswith("out_b"))):
        rng.raw()
    batches = make_batches(tr.all_windows(), tr.series_ids(), 16, prof.horizon, rng)
    order = [(r, a) for b in batches for r, a in zip(b.series_rows, b.anchors)]
    assert order == tr.last_epoch_windows()


def test_oracle_zero_network_validate(oracle):
    """test_trainer.cpp:200-216"""
    prof, vals, cats = dataset(oracle, "tiny", 3, 23)
    tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=16), api=oracle)
    tr.set_weights(np.zeros(tr.n_values))
    v = tr.validate()
    assert np.all(v.forecasts == 0.0) and abs(v.mean_smape - 200.0) < 1e-12


def test_config_validation(oracle):
    """test_trainer.cpp:309-325 through the ABI (ConfigError)."""
    prof, vals, cats = dataset(oracle, "tiny", 2, 1)
    for bad in (dict(tau=1.5), dict(batch_size=4096), dict(gradient_clip=-1.0)):
        with pytest.raises(E.ConfigError):
            Trainer((vals, cats), prof, TrainConfig(**bad), api=oracle)
    with pytest.raises(E.InsufficientLengthError):
        Trainer((vals[:, :10], cats), prof, TrainConfig(), api=oracle)


@pytest.mark.parametrize("name,n,seed", [("quarterly", 8, 9), ("yearly", 20, 2), ("monthly", 5, 3)])
@pytest.mark.parametrize("against_test", [True, False])
def test_oracle_evaluate_matches_reference(oracle, ref, name, n, seed, against_test):
    """cmd_evaluate scoring (commands.hpp:285-338): model and seasonal-naive sMAPE / MASE per
    series, the oracle restatement against the reference's own metrics.hpp functions."""
    prof, vals, cats = dataset(ref, name, n, seed)
    cfg = TrainConfig(seed=seed, batch_size=32)
    o, r = (Trainer((vals, cats), prof, cfg, api=a) for a in (oracle, ref))
    o.train_epoch(), r.train_epoch()
    eo, er = o.evaluate(against_test), r.evaluate(against_test)
    for f in ("forecasts", "smape", "mase", "naive_smape", "naive_mase", "totals"):
        a, b = getattr(eo, f), getattr(er, f)
        assert np.array_equal(np.isnan(a), np.isnan(b)), f
        assert tensor_err(np.nan_to_num(a), np.nan_to_num(b)) < 1e-11, f
    assert eo.model.smape_by_category.keys() == er.model.smape_by_category.keys()
    if not against_test:
        assert max_rel(eo.mean_smape, o.validate().mean_smape) < 1e-14  # validate == evaluate(validation)


def test_mase_undefined_for_periodic_insample(oracle, ref):
    """metrics.hpp:46: a perfectly periodic in-sample span has a zero seasonal-naive MAE, so
    MASE is undefined (std::nullopt -> NaN) and excluded from the aggregates."""
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    cyc = [10.0, 12.0, 9.0, 11.0]
    vals = np.array([cyc * 22, [v * (1 + 0.01 * i) for i, v in enumerate(cyc * 22)]])
    for api in (oracle, ref):
        tr = Trainer((vals, np.array([0, 1], dtype=np.int32)), prof, TrainConfig(seed=1), api=api)
        ev = tr.evaluate(True)
        assert np.isnan(ev.naive_mase[0]) and np.isnan(ev.mase[0]) and not np.isnan(ev.mase[1])
        assert ev.naive_smape[0] == 0.0  # the naive forecast repeats the exact cycle
        assert ev.model.mase_undefined_count == 1 and ev.totals[2] == 1
