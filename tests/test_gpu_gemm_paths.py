"""K3's weight-gradient contraction without the tensor cores has two block shapes: the default
16 x 8 output tiles (TMA-staged row chunks) and the opt-in q-strip blocks (ESRNN_GEMM_WIDE=1,
finish.cuh dw_wide_block: 32 rows of G over all K, row parts combined in part order).  Both
must meet the north-star fp32 contract against the fp64 oracle (pinball kinks masked, as in
test_gpu_fp32_contract.py), agree with each other, and be run-to-run deterministic.
Reference: the MatMul adjoints of Tape::backward (matrix.hpp:103-168, autodiff.hpp:476-482)."""
import numpy as np
import pytest

from conftest import dataset, tensor_err
from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _grads(engine, prof, vals, cats, rows, anchors, mask, B):
    tr = Trainer((vals, cats), prof, TrainConfig(precision="fp32", batch_size=B, seed=7), api=engine)
    return tr.batch_gradients(WindowBatch(rows, anchors, mask=mask.copy()))


@pytest.mark.parametrize("name,n,B", [("quarterly", 400, 1000), ("monthly", 300, 2048)])
def test_q_strip_and_tile_gemm_meet_contract_and_agree(engine, oracle, monkeypatch, name, n, B):
    prof, vals, cats = dataset(oracle, name, n, 23)
    o = Trainer((vals, cats), prof, TrainConfig(precision="fp64", batch_size=B, seed=7), api=oracle)
    w = o.all_windows()
    idx = np.random.default_rng(3).choice(len(w), size=B, replace=False)
    rows, anchors = [w[i][0] for i in idx], [w[i][1] for i in idx]
    b = WindowBatch(rows, anchors)
    o.batch_loss(b)
    pred = o.forward_stack(b.inputs[None])
    mask = np.ones_like(b.targets)
    mask[np.abs(b.targets - pred) < 1e-5] = 0.0
    go = o.batch_gradients(WindowBatch(rows, anchors, mask=mask.copy()))
    monkeypatch.delenv("ESRNN_GEMM_WIDE", raising=False)
    gt = _grads(engine, prof, vals, cats, rows, anchors, mask, B)
    monkeypatch.setenv("ESRNN_GEMM_WIDE", "1")
    gw = _grads(engine, prof, vals, cats, rows, anchors, mask, B)
    gw2 = _grads(engine, prof, vals, cats, rows, anchors, mask, B)
    for k, v in go.network.items():
        assert tensor_err(gt.network[k], v) < TOL, (k, "tiles")
        assert tensor_err(gw.network[k], v) < TOL, (k, "q-strips")
        assert tensor_err(gw.network[k], gt.network[k]) < 1e-5, k
        assert np.array_equal(gw.network[k], gw2.network[k]), k  # fixed summation order
    assert gw.loss == gt.loss


def test_two_tile_ctas_are_bit_identical(engine, oracle, monkeypatch):
    """k_tile<..., NG = 2> (two tiles per CTA on one resident weight copy, chosen for multi-wave
    fp32 steps) runs the same per-tile arithmetic as one tile per CTA: bit-identical epochs."""
    prof, vals, cats = dataset(oracle, "quarterly", 400, 29)
    kw = dict(precision="fp32", batch_size=2048, seed=7, use_graphs=True)
    out = []
    for g2 in ("1", "0"):
        monkeypatch.setenv("ESRNN_TILE_G2", g2)
        tr = Trainer((vals, cats), prof, TrainConfig(**kw), api=engine)
        losses = [tr.train_epoch() for _ in range(2)]
        out.append((losses, tr.weights(), tr.validate().mean_smape))
    assert out[0][0] == out[1][0]
    for k in out[0][1]:
        assert np.array_equal(out[0][1][k], out[1][1][k]), k
    assert out[0][2] == out[1][2]
