#!/usr/bin/env python3
"""fp32 per-step parity probe at the BASELINE batch shapes (cfg1 / cfg2 / cfg3).

For a few sampled batches, the fp32 engine's loss, network gradients (per named array) and
per-series gradients (per parameter kind: alpha_raw, gamma_raw, seasonality_raw) are compared
with the fp64 reference (oracle/_ref, else the C oracle), tensor-scaled (max |a-b| / max |b|),
with and without excluding the pinball kinks: entries whose fp64 |target - prediction| falls
below delta get mask 0 on both sides (the adjoint of |d| jumps by 1/M at d = 0, so
an fp32 rounding that flips the sign of a near-zero d moves the gradient by a whole term).

    python tools/parity_probe.py [cfg1 cfg2 cfg3] > gpurun_out/parity_probe.json
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import ORACLE_LIB, REF_LIB, tensor_err  # noqa: E402
from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer, WindowBatch  # noqa: E402

CFG = {"cfg1": (Frequency.Quarterly, 1000, 88, 4, 1000), "cfg2": (Frequency.Yearly, 23000, 25, 1, 2048),
       "cfg3": (Frequency.Monthly, 48000, 108, 12, 2048)}


def kink_mask(ref_tr, batch, delta):
    """Mask with the pinball kinks removed: |t - p| < delta in the fp64 reference's own
    normalised targets and predictions (its forward_stack on its WindowBatch inputs)."""
    b = WindowBatch(list(batch.series_rows), list(batch.anchors), mask=None)
    ref_tr.batch_loss(b)
    pred = ref_tr.forward_stack(b.inputs[None])
    m = np.ones_like(b.targets) if batch.mask is None else batch.mask.copy()
    near = np.abs(b.targets - pred) < delta
    m[near] = 0.0
    return m, int(near.sum())


def errs(gg, go):
    out = {"loss": abs(gg.loss - go.loss) / abs(go.loss)}
    net = {k: tensor_err(gg.network[k], v) for k, v in go.network.items() if np.any(v)}
    out["net_max"] = max(net.values())
    out["net_worst"] = max(net, key=net.get)
    sids = list(go.per_series)
    for kind, f in (("alpha", lambda p: [p.alpha_raw]), ("gamma", lambda p: [p.gamma_raw]),
                    ("seas", lambda p: list(p.init_seasonality_raw))):
        a = np.concatenate([f(gg.per_series[s]) for s in sids])
        b = np.concatenate([f(go.per_series[s]) for s in sids])
        out["ps_" + kind] = tensor_err(a, b)
        # per-series scaling (the old, stricter-per-row metric), for information
    out["ps_row_max"] = max(
        np.max(np.abs(np.r_[gg.per_series[s].alpha_raw, gg.per_series[s].gamma_raw, gg.per_series[s].init_seasonality_raw]
                      - np.r_[go.per_series[s].alpha_raw, go.per_series[s].gamma_raw, go.per_series[s].init_seasonality_raw]))
        / max(np.max(np.abs(np.r_[go.per_series[s].alpha_raw, go.per_series[s].gamma_raw,
                                  go.per_series[s].init_seasonality_raw])), 1e-300) for s in sids)
    return out


def main():
    names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]
    eng = N.product_api()
    ref_lib = REF_LIB if REF_LIB.exists() else ORACLE_LIB
    ref = N.NativeApi(ref_lib)
    res = {"ref": ref_lib.name}
    for name in names:
        freq, n, length, s, B = CFG[name]
        prof = FrequencyProfile.defaults(freq)
        vals, cats = ref.make_synthetic(41, n, length, s, 0.05)
        g = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp32"), api=eng)
        o = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp64"), api=ref)
        w = o.all_windows()
        rows = []
        # batches 0-1 at the initial state; batches 2-3 after 3 epochs of fp64 engine training
        # (its weights and per-series parameters copied into both trainers): a realistic
        # density of near-kink entries
        for bi in range(4):
            if bi == 2:
                t64 = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp64"), api=eng)
                for _ in range(3):
                    t64.train_epoch()
                wf, (pa, pg, ps) = t64.weights_flat(), t64.per_series_arrays()
                for tr in (g, o):
                    tr.set_weights(wf)
                    tr.set_per_series_arrays(pa, pg, ps)
                t64.close()
            rng = np.random.default_rng(100 + bi)
            idx = rng.choice(len(w), size=B, replace=False)
            base = WindowBatch([w[i][0] for i in idx], [w[i][1] for i in idx])
            rec = {}
            for delta in (0.0, 1e-6, 1e-5, 1e-4, 1e-3):
                if delta == 0.0:
                    m, nk = None, 0
                else:
                    m, nk = kink_mask(o, base, delta)
                bg = WindowBatch(list(base.series_rows), list(base.anchors), mask=None if m is None else m.copy())
                bo = WindowBatch(list(base.series_rows), list(base.anchors), mask=None if m is None else m.copy())
                e = errs(g.batch_gradients(bg), o.batch_gradients(bo))
                e["kinks"] = nk
                e["inputs"] = tensor_err(bg.inputs, bo.inputs)
                e["targets"] = tensor_err(bg.targets, bo.targets)
                rec[str(delta)] = e
            rows.append(rec)
            print(name, bi, json.dumps(rec), file=sys.stderr, flush=True)
        res[name] = rows
    print(json.dumps(res))


if __name__ == "__main__":
    main()
