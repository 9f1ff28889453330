"""The tensor-core weight-gradient path (K3 on steps of >= 4,096 windows, fp32): tcgen05.mma
kind::tf32 with a 3xTF32 split (csrc/umma.cuh, finish.cuh dw_umma_block), against the fp64
oracle at the north-star 1e-4 (pinball kinks masked on both sides, as in
test_gpu_fp32_contract.py), against the CUDA-core path (ESRNN_NO_UMMA), and for determinism.
Reference: the contractions of Tape::backward's MatMul adjoints (matrix.hpp:103-168,
autodiff.hpp:476-482)."""
import numpy as np
import pytest

from conftest import dataset, max_rel, tensor_err
from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _batch(tr, B, seed):
    w = tr.all_windows()
    idx = np.random.default_rng(seed).choice(len(w), size=B, replace=False)
    return [w[i][0] for i in idx], [w[i][1] for i in idx]


def _kink_mask(o, rows, anchors, delta=1e-5):
    b = WindowBatch(list(rows), list(anchors))
    o.batch_loss(b)
    pred = o.forward_stack(b.inputs[None])
    m = np.ones_like(b.targets)
    m[np.abs(b.targets - pred) < delta] = 0.0
    return m


@pytest.mark.parametrize("name,n,B", [("monthly", 300, 8500), ("quarterly", 240, 12000)])
def test_umma_gradients_within_contract(engine, oracle, name, n, B):
    prof, vals, cats = dataset(oracle, name, n, 17)
    kw = dict(batch_size=B, max_batch_size=16384, seed=7)
    g = Trainer((vals, cats), prof, TrainConfig(precision="fp32", **kw), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(precision="fp64", **kw), api=oracle)
    rows, anchors = _batch(o, B, 5)
    m = _kink_mask(o, rows, anchors)
    assert (m == 0).mean() < 5e-3
    gg = g.batch_gradients(WindowBatch(rows, anchors, mask=m.copy()))
    go = o.batch_gradients(WindowBatch(rows, anchors, mask=m.copy()))
    errs = {"loss": abs(gg.loss - go.loss) / abs(go.loss)}
    for k, v in go.network.items():
        errs[k] = tensor_err(gg.network[k], v)
    sids = list(go.per_series)
    errs["ps"] = tensor_err(np.concatenate([[gg.per_series[s].alpha_raw, gg.per_series[s].gamma_raw,
                                             *gg.per_series[s].init_seasonality_raw] for s in sids]),
                            np.concatenate([[go.per_series[s].alpha_raw, go.per_series[s].gamma_raw,
                                             *go.per_series[s].init_seasonality_raw] for s in sids]))
    print(name, {k: f"{v:.2e}" for k, v in errs.items()})
    assert max(errs.values()) < TOL, errs


def test_umma_matches_cuda_core_path_and_is_deterministic(engine, oracle, monkeypatch):
    prof, vals, cats = dataset(oracle, "monthly", 300, 17)
    kw = dict(batch_size=8500, max_batch_size=16384, seed=7, precision="fp32")
    rows, anchors = _batch(Trainer((vals, cats), prof, TrainConfig(**kw), api=oracle), 8500, 9)
    t1 = Trainer((vals, cats), prof, TrainConfig(**kw), api=engine)
    t2 = Trainer((vals, cats), prof, TrainConfig(**kw), api=engine)
    monkeypatch.setenv("ESRNN_NO_UMMA", "1")
    tf = Trainer((vals, cats), prof, TrainConfig(**kw), api=engine)  # CUDA-core (FFMA) GEMM
    monkeypatch.delenv("ESRNN_NO_UMMA")
    g1, g2, gf = (t.batch_gradients(WindowBatch(rows, anchors)) for t in (t1, t2, tf))
    for k in g1.network:
        assert np.array_equal(g1.network[k], g2.network[k]), k          # bit-deterministic
        assert tensor_err(g1.network[k], gf.network[k]) < 2e-5, k       # same contraction
    assert g1.loss == gf.loss  # K2 is shared: identical forward


def test_umma_training_epoch_tracks_oracle(engine, oracle):
    prof, vals, cats = dataset(oracle, "quarterly", 200, 3)
    kw = dict(batch_size=8192, max_batch_size=16384, seed=11)
    g = Trainer((vals, cats), prof, TrainConfig(precision="fp32", **kw), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(precision="fp64", **kw), api=oracle)
    for _ in range(2):
        assert max_rel(g.train_epoch(), o.train_epoch()) < 1e-3
    assert tensor_err(g.weights_flat(), o.weights_flat()) < 1e-3
