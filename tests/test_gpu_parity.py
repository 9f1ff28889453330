"""GPU parity: the CUDA engine (through the C-ABI) against the fp64 C oracle on identical
seeded inputs.  fp64 mode must agree to ~1e-10; fp32 mode carries the north-star
contract of 1e-4 relative per step (tensor-scaled, see tensor_err).

Mirrors the reference's own checks: batched window elements / loss (acceptance.cpp:332-373),
joint gradients (test_trainer.cpp:139-161), masking (acceptance.cpp:493-550), updates
(test_trainer.cpp:96-137), forecast/validate (test_trainer.cpp:200-216), determinism
(test_trainer.cpp:218-230).
"""
import numpy as np
import pytest

from conftest import PROFILES, dataset, max_rel, tensor_err
from paper_1907_03329_b200 import errors as E
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer, WindowBatch

pytestmark = pytest.mark.gpu

CASES = [("tiny", 3, 11, 16), ("quarterly", 12, 41, 64), ("yearly", 40, 5, 64), ("monthly", 9, 7, 64)]


def pair(engine, oracle, name, n, seed, precision="fp64", **kw):
    prof, vals, cats = dataset(oracle, name, n, seed)
    cfg = TrainConfig(seed=7, precision=precision, **kw)
    return (Trainer((vals, cats), prof, cfg, api=engine), Trainer((vals, cats), prof, cfg, api=oracle))


def sample_batch(tr, B, seed, masked_rows=(), partial_row=None):
    rng = np.random.default_rng(seed)
    w = tr.all_windows()
    idx = rng.integers(0, len(w), size=B)
    O = tr.profile().horizon
    mask = np.ones((B, O))
    for r in masked_rows:
        mask[r] = 0.0
    if partial_row is not None:
        mask[partial_row, ::2] = 0.0
    return WindowBatch([w[i][0] for i in idx], [w[i][1] for i in idx], mask=mask)


def copy_batch(b):
    return WindowBatch(list(b.series_rows), list(b.anchors), mask=None if b.mask is None else b.mask.copy())


@pytest.mark.parametrize("name,n,seed,B", CASES)
def test_init_weights_identical(engine, oracle, name, n, seed, B):
    g, o = pair(engine, oracle, name, n, seed)
    assert np.array_equal(g.weights_flat(), o.weights_flat())  # same RNG consumption (network.hpp:89-116)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-4)])
@pytest.mark.parametrize("name,n,seed,B", CASES)
def test_batch_gradients(engine, oracle, name, n, seed, B, precision, tol):
    g, o = pair(engine, oracle, name, n, seed, precision)
    b = sample_batch(o, B, seed, masked_rows=(1,), partial_row=2)
    bg, bo = copy_batch(b), copy_batch(b)
    gg, go = g.batch_gradients(bg), o.batch_gradients(bo)
    assert max_rel(gg.loss, go.loss) < tol
    for f in ("inputs", "targets", "seasonality_slices", "anchor_levels"):
        assert tensor_err(getattr(bg, f), getattr(bo, f)) < tol, f
    assert gg.slot_rows == go.slot_rows
    for name_, arr in go.network.items():
        assert tensor_err(gg.network[name_], arr) < tol * 10, name_
        if name_.endswith("w_recur"):
            assert not np.any(gg.network[name_])  # structurally zero at sequence length 1
    for sid, ps in go.per_series.items():
        pg = gg.per_series[sid]
        v_g = np.r_[pg.alpha_raw, pg.gamma_raw, pg.init_seasonality_raw]
        v_o = np.r_[ps.alpha_raw, ps.gamma_raw, ps.init_seasonality_raw]
        scale = max(np.max(np.abs(v_o)), 1e-12)
        assert np.max(np.abs(v_g - v_o)) / scale < tol * 100, sid


@pytest.mark.parametrize("name,n,seed,B", CASES[:2])
def test_loss_only_matches(engine, oracle, name, n, seed, B):
    g, o = pair(engine, oracle, name, n, seed)
    b = sample_batch(o, B, seed + 1)
    assert max_rel(g.batch_loss(copy_batch(b)), o.batch_loss(copy_batch(b))) < 1e-12


@pytest.mark.parametrize("name,n,seed,bs", [("tiny", 3, 11, 16), ("quarterly", 10, 41, 64),
                                            ("yearly", 60, 5, 32), ("monthly", 6, 7, 48)])
def test_train_epochs_fp64_trajectory(engine, oracle, name, n, seed, bs):
    g, o = pair(engine, oracle, name, n, seed, batch_size=bs)
    for _ in range(2):
        lg, lo = g.train_epoch(), o.train_epoch()
        assert max_rel(lg, lo) < 1e-8
    assert tensor_err(g.weights_flat(), o.weights_flat()) < 1e-7
    ag, gg_, sg = g.per_series_arrays()
    ao, go_, so = o.per_series_arrays()
    assert tensor_err(np.c_[ag, gg_, sg], np.c_[ao, go_, so]) < 1e-7
    vg, vo = g.validate(), o.validate()
    assert max_rel(vg.mean_smape, vo.mean_smape) < 1e-8
    assert tensor_err(vg.forecasts, vo.forecasts) < 1e-8


def test_train_epoch_fp32_tracks_oracle(engine, oracle):
    g, o = pair(engine, oracle, "quarterly", 10, 41, "fp32", batch_size=64)
    lg, lo = g.train_epoch(), o.train_epoch()
    assert max_rel(lg, lo) < 1e-3
    assert abs(g.validate().mean_smape - o.validate().mean_smape) < 0.1


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", ["tiny", "quarterly", "yearly", "monthly"])
def test_forecast_at(engine, oracle, name, precision):
    prof = PROFILES[name][0]
    g, o = pair(engine, oracle, name, 7, 3, precision)
    tol = 1e-12 if precision == "fp64" else 1e-5
    for drop in (0, prof.horizon, 2 * prof.horizon):
        assert tensor_err(g.forecast_at(drop).forecasts, o.forecast_at(drop).forecasts) < tol


def test_hw_state_matches_oracle(engine, oracle):
    g, o = pair(engine, oracle, "monthly", 4, 3)
    a = np.array([0.3, -0.7, 1.1, 2.0])
    s = np.linspace(-0.2, 0.2, 4 * 12).reshape(4, 12)
    for t in (g, o):
        t.set_per_series_arrays(a, -a, s)
    for row in range(4):
        for tl in (12, 50, 108):
            lg, sg = g.hw_state(row, tl)
            lo, so = o.hw_state(row, tl)
            assert max_rel(lg, lo) < 1e-13 and max_rel(sg, so) < 1e-13


def test_masking_bit_zero(engine, oracle):
    """acceptance.cpp:493-550: padded rows with mask 0 give bit-zero per-series gradients."""
    g, _ = pair(engine, oracle, "quarterly", 6, 71)
    I, O = 12, 8
    small = WindowBatch([0, 1, 2, 3], [I - 1, I + 5, I + 9, I + 2], mask=np.ones((4, O)))
    padded = WindowBatch([0, 1, 2, 3, 4, 5], [I - 1, I + 5, I + 9, I + 2, I + 7, I + 1], mask=np.ones((6, O)))
    padded.mask[4:] = 0.0
    gs, gp = g.batch_gradients(small), g.batch_gradients(padded)
    assert abs(gs.loss - gp.loss) <= 1e-12
    for k, v in gs.network.items():
        assert np.max(np.abs(v - gp.network[k])) <= 1e-12
    for sid in ("S4", "S5"):
        p = gp.per_series[sid]
        assert p.alpha_raw == 0.0 and p.gamma_raw == 0.0 and not np.any(p.init_seasonality_raw)


def test_zero_learning_rates_bit_unchanged(engine, oracle):
    """test_trainer.cpp:96-119"""
    g, _ = pair(engine, oracle, "tiny", 3, 11, batch_size=16, learning_rate_network=0.0,
                learning_rate_per_series=0.0)
    w0 = g.weights_flat()
    p0 = g.per_series_arrays()
    assert np.isfinite(g.train_epoch())
    assert np.array_equal(w0, g.weights_flat())
    for a, b in zip(p0, g.per_series_arrays()):
        assert np.array_equal(a, b)


def test_detached_state_freezes_per_series(engine, oracle):
    """test_trainer.cpp:274-282"""
    g, o = pair(engine, oracle, "tiny", 2, 41, batch_size=16, attach_es_state=False)
    p0 = g.per_series_arrays()
    lg, lo = g.train_epoch(), o.train_epoch()
    assert max_rel(lg, lo) < 1e-9
    for a, b in zip(p0, g.per_series_arrays()):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_same_seed_bit_identical(engine, oracle, precision):
    """test_trainer.cpp:218-230: same seed reproduces the loss trajectory bit for bit."""
    a, _ = pair(engine, oracle, "quarterly", 20, 29, precision, batch_size=64)
    b, _ = pair(engine, oracle, "quarterly", 20, 29, precision, batch_size=64)
    for _ in range(3):
        assert a.train_epoch() == b.train_epoch()
    assert a.validate().mean_smape == b.validate().mean_smape


def test_validate_zero_network(engine, oracle):
    """test_trainer.cpp:200-216: zero weights -> forecasts 0, sMAPE 200, read-only."""
    g, _ = pair(engine, oracle, "tiny", 3, 23)
    g.set_weights(np.zeros(g.n_values))
    v1, v2 = g.validate(), g.validate()
    assert np.all(v1.forecasts == 0.0)
    assert abs(v1.mean_smape - 200.0) < 1e-12
    assert v1.mean_smape == v2.mean_smape


def test_errors(engine, oracle):
    g, _ = pair(engine, oracle, "tiny", 3, 11)
    with pytest.raises(E.ShapeError):
        g.batch_loss(WindowBatch([0], [100]))
    with pytest.raises(E.ContractError):
        g.batch_loss(WindowBatch([0], [7], mask=np.zeros((1, 4))))
    with pytest.raises(E.ContractError):
        g.batch_loss(WindowBatch([], []))
    with pytest.raises(E.CheckpointError):
        g.set_weights(np.zeros(3))
    with pytest.raises(E.InsufficientLengthError):
        g.forecast_at(1000)


def test_numeric_domain_error(engine, oracle):
    prof, vals, cats = dataset(oracle, "tiny", 2, 5)
    vals[1, 3] = -vals[1, 3] * 50.0  # drives a level negative mid-scan
    g = Trainer((vals, cats), prof, TrainConfig(seed=1, batch_size=16), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(seed=1, batch_size=16), api=oracle)
    with pytest.raises(E.NumericDomainError):
        o.train_epoch()
    with pytest.raises(E.NumericDomainError):
        g.train_epoch()
    with pytest.raises(E.NumericDomainError):
        g.validate()


# ------------------------------------------------------------------ reference goldens
import golden_check  # noqa: E402


@pytest.mark.parametrize("name", golden_check.FIXTURES)
def test_engine_matches_reference_golden_fp64(engine, name):
    """Replays the reference-generated fixture: init weights, one masked batch (loss,
    WindowBatch matrices, slot order, all gradients), two epochs (losses, bit-exact window
    order, parameters), validate / forecast_at(0), post-training HW state."""
    golden_check.check(engine, name, "fp64", tol=1e-10, tol_train=1e-9)


@pytest.mark.parametrize("name", golden_check.FIXTURES)
def test_engine_matches_reference_golden_fp32_step(engine, name):
    """fp32 performance mode against the same fixture: first-step losses/gradients within
    the north-star 1e-4 (tensor-scaled), window order still bit-exact."""
    fx = golden_check.load(name)
    prof = PROFILES[fx["profile"]][0]
    tr = Trainer((np.array(fx["values"]), np.array(fx["categories"], dtype=np.int32)), prof,
                 TrainConfig(seed=fx["train_seed"], batch_size=fx["batch_size"], precision="fp32"), api=engine)
    bt = fx["batch"]
    b = WindowBatch(list(bt["rows"]), list(bt["anchors"]), mask=np.array(bt["mask"]))
    g = tr.batch_gradients(b)
    assert abs(g.loss - bt["loss"]) <= 1e-4 * abs(bt["loss"])
    for k, v in bt["net_grads"].items():
        golden_check._cmp_array(g.network[k], v, 1e-3, k)
    tr.train_epoch()
    tr.train_epoch()
    assert [list(x) for x in tr.last_epoch_windows()[:512]] == fx["last_epoch_windows"]


# ------------------------------------------------------------------ window indices
def test_epoch_window_order_bit_exact_vs_reference(engine, oracle):
    """North-star contract: bit-exact window indices.  The engine's host replica of
    all_windows + Rng::shuffle equals the reference / oracle order, epoch after epoch."""
    from conftest import REF_LIB
    from paper_1907_03329_b200._native import NativeApi
    apis = [oracle] + ([NativeApi(REF_LIB)] if REF_LIB.exists() else [])
    prof, vals, cats = dataset(oracle, "quarterly", 30, 3)
    trs = [Trainer((vals, cats), prof, TrainConfig(seed=99, batch_size=100), api=a) for a in [engine] + apis]
    for _ in range(3):
        orders = []
        for t in trs:
            t.train_epoch()
            orders.append(t.last_epoch_windows())
        assert all(o == orders[0] for o in orders[1:])


# ------------------------------------------------------------------ sharded data path
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_sharded_partials_sum_to_full_batch(engine, oracle, world, precision):
    """Series-sharded ranks on one GPU (local-partials mode: the data path of every rank
    runs, the collective is summed here): the per-rank partial loss / shared gradients add
    up to the single-GPU step; per-series gradients stay with their owner."""
    from sharding_helpers import LOCAL_PARTIALS_ID, shard_range
    prof, vals, cats = dataset(oracle, "monthly", 10, 4)
    cfg = TrainConfig(seed=7, batch_size=64, precision=precision)
    full = Trainer((vals, cats), prof, cfg, api=engine)
    b = sample_batch(full, 64, 5, masked_rows=(3,))
    gf = full.batch_gradients(copy_batch(b))
    tot_loss, tot = 0.0, {k: np.zeros_like(v) for k, v in gf.network.items()}
    for r in range(world):
        tr = Trainer((vals, cats), prof, cfg, api=engine, dist=(r, world, LOCAL_PARTIALS_ID))
        assert (tr.row_begin, tr.row_end) == shard_range(r, world, 10)
        g = tr.batch_gradients(copy_batch(b))
        tot_loss += g.loss
        for k in tot:
            tot[k] += g.network[k]
        for sid, p in g.per_series.items():
            assert tr.row_begin <= int(sid[1:]) < tr.row_end
            ref = gf.per_series[sid]
            scale = max(abs(ref.alpha_raw), abs(ref.gamma_raw), np.max(np.abs(ref.init_seasonality_raw)))
            tol = 1e-9 if precision == "fp64" else 1e-3
            assert abs(p.alpha_raw - ref.alpha_raw) <= tol * scale
    tol = 1e-12 if precision == "fp64" else 1e-5
    assert abs(tot_loss - gf.loss) <= tol * abs(gf.loss)
    for k, v in gf.network.items():
        assert tensor_err(tot[k], v) <= (1e-11 if precision == "fp64" else 1e-4), k


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-5)])
@pytest.mark.parametrize("name", ["quarterly", "yearly", "monthly"])
@pytest.mark.parametrize("against_test", [True, False])
def test_evaluate_scores(engine, oracle, name, precision, tol, against_test):
    """Device-side cmd_evaluate scoring (sMAPE, MASE, seasonal-naive) vs the oracle."""
    g, o = pair(engine, oracle, name, 37, 4, precision, batch_size=64)
    for tr in (g, o):
        tr.train_epoch()
    eg, eo = g.evaluate(against_test), o.evaluate(against_test)
    for f in ("forecasts", "smape", "mase", "naive_smape", "naive_mase"):
        a, b = getattr(eg, f), getattr(eo, f)
        assert np.array_equal(np.isnan(a), np.isnan(b)), f
        assert tensor_err(np.nan_to_num(a), np.nan_to_num(b)) < (tol if "naive" not in f else 1e-6), f
    assert abs(eg.mean_smape - eo.mean_smape) < 100 * tol
    assert abs(eg.mean_mase - eo.mean_mase) < 100 * tol


def test_quality_parity_cfg1_15_epochs(engine, ref):
    """North-star quality contract: after the same 15 epochs and seeds on cfg1 (Quarterly,
    1,000 series, B=1,000), the fp32 engine's holdout sMAPE and MASE are within 0.1 of the
    reference's own fp64 CPU run (oracle/_ref).  Trajectories diverge chaotically at fp32
    (SURVEY §7 hard parts), so only end-of-run quality is compared."""
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    vals, cats = ref.make_synthetic(41, 1000, 88, 4, 0.05)
    scores = {}
    for key, api, prec in (("gpu", engine, "fp32"), ("ref", ref, "fp64")):
        tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=1000, precision=prec), api=api)
        for _ in range(15):
            tr.train_epoch()
        v = tr.evaluate(False)
        t = tr.evaluate(True)
        scores[key] = (v.mean_smape, v.mean_mase, t.mean_smape, t.mean_mase)
    g, r = scores["gpu"], scores["ref"]
    assert all(abs(a - b) < 0.1 for a, b in zip(g, r)), (g, r)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_two_live_trainers_interleaved_bit_identical(engine, oracle, precision):
    """Two trainers of the same configuration alive at once, epochs interleaved: the shared
    process-wide caches (device / pinned blocks, epoch graphs, plan worker pool) must not
    couple them (test_trainer.cpp:218-230 determinism, with the C++ API's usage pattern)."""
    prof, vals, cats = dataset(oracle, "quarterly", 9, 29)
    cfg = TrainConfig(seed=42, batch_size=32, precision=precision)
    t1 = Trainer((vals, cats), prof, cfg, api=engine)
    t2 = Trainer((vals, cats), prof, cfg, api=engine)
    for _ in range(4):
        assert t1.train_epoch() == t2.train_epoch()
        assert t1.last_epoch_windows() == t2.last_epoch_windows()
    assert np.array_equal(t1.weights_flat(), t2.weights_flat())
    assert t1.validate().mean_smape == t2.validate().mean_smape


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("fp64", 1e-10)])
def test_two_wave_batch_matches_oracle(engine, oracle, precision, tol):
    """A batch of more than two waves of 8-window tiles (>= 2 x 148 x 8 windows) runs the
    staged two-CTAs-per-SM tile variant: same loss and gradients as the oracle."""
    prof, vals, cats = dataset(oracle, "monthly", 90, 13)
    kw = dict(batch_size=2400, max_batch_size=4096)
    g = Trainer((vals, cats), prof, TrainConfig(seed=7, precision=precision, **kw), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(seed=7, precision="fp64", **kw), api=oracle)
    b = sample_batch(o, 2400, 3)
    gg, go = g.batch_gradients(copy_batch(b)), o.batch_gradients(copy_batch(b))
    assert max_rel(gg.loss, go.loss) < tol
    for name_, arr in go.network.items():
        assert tensor_err(gg.network[name_], arr) < tol * 10, name_
    lg, lo = g.train_epoch(), o.train_epoch()
    assert max_rel(lg, lo) < (1e-8 if precision == "fp64" else 1e-3)


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-4), ("fp64", 1e-10)])
def test_large_step_split_gradient_tiles(engine, oracle, precision, tol):
    """A step of >= 8,192 windows splits each weight-gradient tile's rows over several blocks
    (ticketed, fixed-order combine): gradients still match the oracle."""
    prof, vals, cats = dataset(oracle, "monthly", 300, 17)
    kw = dict(batch_size=8500, max_batch_size=16384)
    g = Trainer((vals, cats), prof, TrainConfig(seed=7, precision=precision, **kw), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(seed=7, precision="fp64", **kw), api=oracle)
    b = sample_batch(o, 8500, 5)
    gg, go = g.batch_gradients(copy_batch(b)), o.batch_gradients(copy_batch(b))
    assert max_rel(gg.loss, go.loss) < tol
    for name_, arr in go.network.items():
        assert tensor_err(gg.network[name_], arr) < tol * 10, name_
    # determinism of the split combine
    g2 = Trainer((vals, cats), prof, TrainConfig(seed=7, precision=precision, **kw), api=engine)
    gg2 = g2.batch_gradients(copy_batch(b))
    for name_ in go.network:
        assert np.array_equal(gg.network[name_], gg2.network[name_]), name_


@pytest.mark.parametrize("freq", [Frequency.Yearly, Frequency.Quarterly, Frequency.Monthly])
def test_forecast_scan_reports_first_bad_observation(engine, oracle, freq):
    """K6 is specialised per season length (S = 1/4/12); its folded error checks must report
    the first non-positive observation, as the reference's scan throws there."""
    prof = FrequencyProfile.defaults(freq)
    length = prof.min_length + 2 * prof.horizon
    vals, cats = oracle.make_synthetic(5, 40, length, prof.seasonality_length, 0.05)
    p = length - 2 * prof.horizon - 3
    vals[17, p] = 0.0
    vals[29, p + 1] = -1.0
    for api in (engine, oracle):
        tr = Trainer((vals, cats), prof, TrainConfig(seed=1, batch_size=64), api=api)
        with pytest.raises(E.NumericDomainError, match=f"t={p}\\b"):
            tr.validate()
