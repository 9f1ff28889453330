#!/usr/bin/env python3
"""Quality goldens: the REFERENCE's own holdout scores after the north-star protocol
(15 epochs, train seed 7, data seed 41) at BASELINE configs[1] (cfg2, M4-Yearly shape,
23,000 series, B = 2,048) and configs[2] (cfg3, M4-Monthly shape, 48,000 series,
B = 2,048), plus the SHA-256 of its shuffled window order for the first two epochs of
cfg3 (1,488,000 windows per epoch; bit-exact window-index contract at full scale).

The reference is oracle/_ref/libesrnn_ref.so (built by oracle/Makefile from
/root/reference/proj/include, unmodified, behind oracle/ref_shim.cpp).  cfg3 takes
~7 minutes of reference CPU time, which is why the scores are recorded here instead of
re-run on the GPU box (tests/test_gpu_fp32_contract.py compares against this file).

    make -C oracle && python tests/golden/make_quality_golden.py [cfg2 cfg3]
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer  # noqa: E402

OUT = Path(__file__).resolve().parent / "quality.json"
CFG = {"cfg1": (Frequency.Quarterly, 1000, 88, 4, 1000), "cfg2": (Frequency.Yearly, 23000, 25, 1, 2048),
       "cfg3": (Frequency.Monthly, 48000, 108, 12, 2048)}
EPOCHS = 15


def order_hash(order) -> str:
    a = np.asarray(order, dtype=np.int32)
    return hashlib.sha256(a.tobytes()).hexdigest()


def run(name):
    freq, n, length, s, B = CFG[name]
    ref = N.NativeApi(ROOT / "oracle" / "_ref" / "libesrnn_ref.so")
    prof = FrequencyProfile.defaults(freq)
    vals, cats = ref.make_synthetic(41, n, length, s, 0.05)
    tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, precision="fp64"), api=ref)
    t0 = time.time()
    losses, hashes = [], []
    for e in range(EPOCHS):
        losses.append(tr.train_epoch())
        if e < 2:
            hashes.append(order_hash(tr.last_epoch_windows()))
        print(name, e, losses[-1], f"{time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    v, t = tr.evaluate(False), tr.evaluate(True)
    return {"series": n, "length": length, "batch_size": B, "epochs": EPOCHS, "data_seed": 41, "train_seed": 7,
            "epoch_losses": losses, "window_order_sha256": hashes,
            "val_smape": v.mean_smape, "val_mase": v.mean_mase, "test_smape": t.mean_smape, "test_mase": t.mean_mase,
            "ref_seconds": time.time() - t0}


def main():
    names = sys.argv[1:] or ["cfg2", "cfg3"]
    doc = json.loads(OUT.read_text()) if OUT.exists() else {}
    doc["generator"] = "tests/golden/make_quality_golden.py (reference: oracle/_ref/libesrnn_ref.so)"
    for name in names:
        doc[name] = run(name)
        OUT.write_text(json.dumps(doc, indent=1) + "\n")


if __name__ == "__main__":
    main()
