"""The opt-in level-variability penalty on the engine against the oracle's restatement
(pinned on CPU in tests/test_penalty.py: closed form, central differences, weight 0 = the
reference).  Fused into K3's ES blocks: its value joins the step's loss sum and its adjoint
the level adjoints of the reverse Holt-Winters scan (paper_1907_03329_b200/csrc/finish.cuh).
"""
import numpy as np
import pytest

from conftest import dataset, max_rel, tensor_err
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch

pytestmark = pytest.mark.gpu
LAM = 3.0


def _trainers(engine, oracle, name, n, seed, prec, B=64, lam=LAM):
    prof, vals, cats = dataset(oracle, name, n, seed)
    g = Trainer((vals, cats), prof, TrainConfig(seed=seed, batch_size=B, precision=prec,
                                                level_variability_penalty=lam), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(seed=seed, batch_size=B, level_variability_penalty=lam), api=oracle)
    return g, o


def _grad_errs(gg, go):
    e = {"loss": abs(gg.loss - go.loss) / abs(go.loss)}
    for k, v in go.network.items():
        e[k] = tensor_err(gg.network[k], v)
    sids = list(go.per_series)
    for kind, f in (("alpha", lambda p: [p.alpha_raw]), ("gamma", lambda p: [p.gamma_raw]),
                    ("seas", lambda p: list(p.init_seasonality_raw))):
        e["ps." + kind] = tensor_err(np.concatenate([f(gg.per_series[s]) for s in sids]),
                                     np.concatenate([f(go.per_series[s]) for s in sids]))
    return e


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-10), ("fp32", 1e-4)])
@pytest.mark.parametrize("name", ["quarterly", "yearly", "monthly"])
def test_penalised_batch_gradients_match_oracle(engine, oracle, name, prec, tol):
    g, o = _trainers(engine, oracle, name, 40, 5, prec)
    w = o.all_windows()
    idx = np.random.default_rng(3).choice(len(w), size=min(96, len(w)), replace=False)
    rows, anchors = [w[i][0] for i in idx], [w[i][1] for i in idx]
    gg, go = g.batch_gradients(WindowBatch(rows, anchors)), o.batch_gradients(WindowBatch(rows, anchors))
    e = _grad_errs(gg, go)
    assert max(e.values()) < tol, e
    # batch_loss (no gradient request) includes the penalty too
    assert max_rel(g.batch_loss(WindowBatch(rows, anchors)), go.loss) < tol


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("fp32", 1e-3)])
def test_penalised_training_matches_oracle(engine, oracle, prec, tol):
    g, o = _trainers(engine, oracle, "quarterly", 60, 7, prec, B=128)
    for _ in range(2):
        assert max_rel(g.train_epoch(), o.train_epoch()) < tol
    assert tensor_err(g.weights_flat(), o.weights_flat()) < tol
    for a, b in zip(g.per_series_arrays(), o.per_series_arrays()):
        assert tensor_err(a, b) < tol


def test_penalty_changes_training(engine, oracle):
    g, _ = _trainers(engine, oracle, "quarterly", 60, 7, "fp64", B=128)
    z, _ = _trainers(engine, oracle, "quarterly", 60, 7, "fp64", B=128, lam=0.0)
    lg, lz = g.train_epoch(), z.train_epoch()
    assert lg > lz  # the penalty adds a positive term
    assert tensor_err(g.per_series_arrays()[0], z.per_series_arrays()[0]) > 1e-6


def test_penalised_group_sharded_matches_single(engine, oracle):
    """world 2 in-process group: the penalty's partials travel in the step's loss sum and the
    per-series gradients stay with their owner."""
    import threading
    prof, vals, cats = dataset(oracle, "quarterly", 50, 9)
    cfg = TrainConfig(seed=9, batch_size=100, precision="fp64", level_variability_penalty=LAM)
    single = Trainer((vals, cats), prof, cfg, api=engine)
    want = [single.train_epoch() for _ in range(2)]
    grp = engine.group(2)
    trs, out = [None, None], [None, None]

    def run(r):
        try:
            trs[r] = Trainer((vals, cats), prof, cfg, api=engine, dist=(r, 2, grp, 0))
            out[r] = [trs[r].train_epoch() for _ in range(2)]
        except Exception as e:  # noqa: BLE001
            out[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for r in range(2):
        assert not isinstance(out[r], Exception), out[r]
        assert max_rel(out[r], want) < 1e-10
    assert tensor_err(trs[0].weights_flat(), single.weights_flat()) < 1e-10
    for t in trs:
        t.close()
    grp.close()
