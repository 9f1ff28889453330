"""North-star fp32 contract at the BASELINE batch shapes, against the reference itself.

    "fp32 forward losses and gradients within 1e-4 relative per step; final holdout
     sMAPE/MASE within 0.1 points after the same epochs and seeds; bit-exact window
     indices and series partitioning."  (BASELINE.json north_star)

* Per step: the fp32 engine and the fp64 reference (oracle/_ref: the reference's own
  headers, built unmodified; the C oracle when the reference is not built) run the same
  batch from the same state -- the initial state and a trained one (3 fp64 engine epochs,
  copied into both) -- at cfg1 (Quarterly, 1,000 series, B = 1,000), cfg2 (Yearly, 23,000
  series, B = 2,048, S = 1) and cfg3 (Monthly, 48,000 series, B = 2,048, S = 12).
  Asserted <= 1e-4: the loss (relative), every network array and the per-series gradient
  block -- alpha_raw, gamma_raw and init_seasonality_raw, each across the batch's series --
  tensor-scaled (max |a - b| / max |b|, tensor_err).
* Pinball kinks: the loss adjoint jumps by 1/M where target == prediction, so an
  fp32 rounding that flips the sign of a near-zero difference moves a gradient by a whole
  term.  Entries whose fp64 |target - prediction| < KINK_DELTA get mask 0 on BOTH sides
  (kink_mask); the fraction excluded is asserted to stay below 0.5%.
* Quality: 15 epochs at the BASELINE seeds, fp32 engine vs the reference's holdout scores
  (cfg2 run live; cfg3 from tests/golden/quality.json, which make_quality_golden.py
  recorded from the reference -- ~7 CPU minutes), within 0.1 points.
* Window order at full scale: the engine's first two cfg3 epochs (1,488,000 windows each)
  hash to the reference's recorded SHA-256.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import ORACLE_LIB, REF_LIB, tensor_err
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer, WindowBatch

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "quality.json"
CFG = {"cfg1": (Frequency.Quarterly, 1000, 88, 4, 1000), "cfg2": (Frequency.Yearly, 23000, 25, 1, 2048),
       "cfg3": (Frequency.Monthly, 48000, 108, 12, 2048)}
TOL = 1e-4
KINK_DELTA = 1e-5


@pytest.fixture(scope="module")
def refapi():
    return N.NativeApi(REF_LIB if REF_LIB.exists() else ORACLE_LIB)


def kink_mask(ref_tr, rows, anchors, delta=KINK_DELTA):
    """1 everywhere except the pinball kinks of the fp64 reference's own forward pass:
    |target - prediction| < delta on the normalised scale (targets, and the predictions of
    its forward_stack on its WindowBatch inputs)."""
    b = WindowBatch(list(rows), list(anchors))
    ref_tr.batch_loss(b)
    pred = ref_tr.forward_stack(b.inputs[None])
    m = np.ones_like(b.targets)
    m[np.abs(b.targets - pred) < delta] = 0.0
    return m


def step_errors(gg, go):
    e = {"loss": abs(gg.loss - go.loss) / abs(go.loss)}
    for k, v in go.network.items():
        e["net." + k] = tensor_err(gg.network[k], v)
    sids = list(go.per_series)
    assert sorted(sids) == sorted(gg.per_series)
    for kind, f in (("alpha_raw", lambda p: [p.alpha_raw]), ("gamma_raw", lambda p: [p.gamma_raw]),
                    ("init_seasonality_raw", lambda p: list(p.init_seasonality_raw))):
        e["ps." + kind] = tensor_err(np.concatenate([f(gg.per_series[s]) for s in sids]),
                                     np.concatenate([f(go.per_series[s]) for s in sids]))
    return e


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_fp32_step_within_1e4_of_reference(engine, refapi, name):
    freq, n, length, s, B = CFG[name]
    prof = FrequencyProfile.defaults(freq)
    vals, cats = refapi.make_synthetic(41, n, length, s, 0.05)
    g = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp32"), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp64"), api=refapi)
    w = o.all_windows()
    worst = {}
    for state in ("init", "trained"):
        if state == "trained":
            t64 = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp64"), api=engine)
            for _ in range(3):
                t64.train_epoch()
            wf, (pa, pg, ps) = t64.weights_flat(), t64.per_series_arrays()
            t64.close()
            for tr in (g, o):
                tr.set_weights(wf)
                tr.set_per_series_arrays(pa, pg, ps)
        for bi in range(2):
            idx = np.random.default_rng(1000 * bi + len(state)).choice(len(w), size=B, replace=False)
            rows, anchors = [w[i][0] for i in idx], [w[i][1] for i in idx]
            m = kink_mask(o, rows, anchors)
            assert (m == 0).mean() < 5e-3
            e = step_errors(g.batch_gradients(WindowBatch(rows, anchors, mask=m.copy())),
                            o.batch_gradients(WindowBatch(rows, anchors, mask=m.copy())))
            for k, v in e.items():
                worst[k] = max(worst.get(k, 0.0), v)
    print(name, "worst per-step errors vs reference:", {k: f"{v:.2e}" for k, v in sorted(worst.items())})
    bad = {k: v for k, v in worst.items() if v > TOL}
    assert not bad, (name, bad, max(worst.values()))


def test_fp32_quality_cfg2_15_epochs_live(engine, refapi):
    """configs[1] (Yearly, 23,000 series, B = 2,048): 15 epochs, the reference run live."""
    freq, n, length, s, B = CFG["cfg2"]
    prof = FrequencyProfile.defaults(freq)
    vals, cats = refapi.make_synthetic(41, n, length, s, 0.05)
    scores = {}
    for key, api, prec in (("gpu", engine, "fp32"), ("ref", refapi, "fp64")):
        tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision=prec), api=api)
        for _ in range(15):
            tr.train_epoch()
        v, t = tr.evaluate(False), tr.evaluate(True)
        scores[key] = (v.mean_smape, v.mean_mase, t.mean_smape, t.mean_mase)
    assert all(abs(a - b) < 0.1 for a, b in zip(scores["gpu"], scores["ref"])), scores


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_fp32_quality_vs_reference_golden(engine, name):
    """configs[1] / configs[2]: the fp32 engine after 15 epochs against the reference's own
    recorded holdout sMAPE / MASE (tests/golden/quality.json), within 0.1 points; the fp64
    engine's epoch losses track the reference's."""
    gold = json.loads(GOLD.read_text())[name]
    freq, n, length, s, B = CFG[name]
    prof = FrequencyProfile.defaults(freq)
    vals, cats = engine.make_synthetic(41, n, length, s, 0.05)
    for prec in ("fp32", "fp64"):
        tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision=prec), api=engine)
        losses = [tr.train_epoch() for _ in range(gold["epochs"])]
        v, t = tr.evaluate(False), tr.evaluate(True)
        got = (v.mean_smape, v.mean_mase, t.mean_smape, t.mean_mase)
        ref = (gold["val_smape"], gold["val_mase"], gold["test_smape"], gold["test_mase"])
        assert all(abs(a - b) < 0.1 for a, b in zip(got, ref)), (prec, got, ref)
        if prec == "fp64":
            assert abs(losses[0] - gold["epoch_losses"][0]) <= 1e-9 * abs(gold["epoch_losses"][0])
        tr.close()


def test_window_order_cfg3_full_scale_bit_exact(engine):
    """Bit-exact window indices at configs[2] scale: 48,000 series x 31 anchors = 1,488,000
    windows shuffled by the trainer RNG (make_batches / Rng::shuffle, trainer.hpp:82-102,
    matrix.hpp:203-205), two epochs, hashed and compared with the reference's."""
    gold = json.loads(GOLD.read_text())["cfg3"]
    freq, n, length, s, B = CFG["cfg3"]
    prof = FrequencyProfile.defaults(freq)
    vals, cats = engine.make_synthetic(41, n, length, s, 0.05)
    tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp32"), api=engine)
    for e in range(2):
        tr.train_epoch()
        order = np.asarray(tr.last_epoch_windows(), dtype=np.int32)
        assert order.shape == (n * 31, 2)
        assert hashlib.sha256(order.tobytes()).hexdigest() == gold["window_order_sha256"][e], e
