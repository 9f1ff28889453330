#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the REFERENCE implementation.

The reference (/root/reference/proj/include, header-only C++) is compiled unmodified
behind oracle/ref_shim.cpp into oracle/_ref/libesrnn_ref.so (oracle/Makefile).  This
script drives it through the same C-ABI the engine exports and records inputs and
outputs as JSON (floats round-trip exactly through repr).  The fixtures pin the
plain-C oracle (tests/test_oracle.py) and travel to the GPU box, where the reference
tree does not exist.

    make -C oracle && python tests/golden/make_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import PROFILES  # noqa: E402
from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch  # noqa: E402

OUT = Path(__file__).resolve().parent
REF = N.NativeApi(ROOT / "oracle" / "_ref" / "libesrnn_ref.so")

# name, profile, n series, data seed, train seed, batch size, full arrays?
CASES = [
    ("tiny", "tiny", 3, 11, 3, 16, True),
    ("quarterly", "quarterly", 8, 41, 7, 64, False),
    ("yearly", "yearly", 24, 5, 7, 32, False),
    ("monthly", "monthly", 5, 7, 7, 48, False),
]
SAMPLE = 24  # sampled entries per large array


def summary(a):
    a = np.asarray(a, dtype=np.float64).ravel()
    idx = np.linspace(0, a.size - 1, min(SAMPLE, a.size)).astype(int)
    return {"n": int(a.size), "sum": float(a.sum()), "l2": float(np.sqrt((a * a).sum())),
            "absmax": float(np.abs(a).max()), "idx": idx.tolist(), "val": a[idx].tolist()}


def main():
    for name, prof_name, n, dseed, tseed, bs, full in CASES:
        prof, length, s, sigma = PROFILES[prof_name]
        vals, cats = REF.make_synthetic(dseed, n, length, s, sigma)
        cfg = TrainConfig(seed=tseed, batch_size=bs, precision="fp64")
        tr = Trainer((vals, cats), prof, cfg, api=REF)
        w0 = tr.weights_flat()
        windows = tr.all_windows()
        rng = np.random.default_rng(dseed)
        idx = rng.integers(0, len(windows), size=bs)
        rows = [windows[i][0] for i in idx]
        anchors = [windows[i][1] for i in idx]
        mask = np.ones((bs, prof.horizon))
        mask[1] = 0.0
        mask[2, ::2] = 0.0
        b = WindowBatch(list(rows), list(anchors), mask=mask.copy())
        g = tr.batch_gradients(b)
        net = {k: (v.ravel().tolist() if full else summary(v)) for k, v in g.network.items()}
        per = {sid: [p.alpha_raw, p.gamma_raw, *p.init_seasonality_raw.tolist()] for sid, p in g.per_series.items()}
        losses = [tr.train_epoch() for _ in range(2)]
        order = tr.last_epoch_windows()
        v = tr.validate()
        f0 = tr.forecast_at(0)
        a, gm, sr = tr.per_series_arrays()
        hw = {str(r): [x.tolist() for x in tr.hw_state(r, length)] for r in range(min(n, 2))}
        fx = {
            "profile": prof_name, "n": n, "length": length, "season": s, "sigma": sigma, "data_seed": dseed,
            "train_seed": tseed, "batch_size": bs, "values": vals.tolist(), "categories": cats.tolist(),
            "init_weights": w0.tolist() if full else summary(w0),
            "batch": {"rows": rows, "anchors": anchors, "mask": mask.tolist(), "loss": g.loss,
                      "inputs": b.inputs.tolist(), "targets": b.targets.tolist(),
                      "seasonality_slices": b.seasonality_slices.tolist(), "anchor_levels": b.anchor_levels.tolist(),
                      "slot_rows": [int(x) for x in g.slot_rows], "net_grads": net, "per_series_grads": per},
            "epoch_losses": losses,
            "last_epoch_windows": order[:512],
            "n_windows": len(order),
            "after_weights": tr.weights_flat().tolist() if full else summary(tr.weights_flat()),
            "after_per_series": {"alpha_raw": a.tolist(), "gamma_raw": gm.tolist(), "seas_raw": sr.tolist()},
            "validate": {"mean_smape": v.mean_smape, "smape": v.smape_per_series.tolist(),
                         "forecasts": v.forecasts.tolist()},
            "forecast_at_0": f0.forecasts.tolist(),
            "hw_state_after": hw,
            "generator": "tests/golden/make_golden.py via oracle/_ref/libesrnn_ref.so (" + REF.version + ")",
        }
        (OUT / f"{name}.json").write_text(json.dumps(fx))
        print("wrote", name, (OUT / f"{name}.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
