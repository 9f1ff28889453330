import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer, WindowBatch
engine = N.product_api(); oracle = N.NativeApi(ROOT / "oracle" / "liboracle_esrnn.so")
prof = FrequencyProfile.defaults(Frequency.Quarterly)
vals, cats = engine.make_synthetic(41, 16, 88, 4, 0.05)
for masked in (False, True):
    g = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=64, precision="fp64"), api=engine)
    o = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=64, precision="fp64"), api=oracle)
    w = g.all_windows()[::7][:64]
    mk = np.ones((64, 8)) if masked else None
    bg = WindowBatch([x[0] for x in w], [x[1] for x in w], mask=mk)
    bo = WindowBatch([x[0] for x in w], [x[1] for x in w], mask=mk)
    gg, go = g.batch_gradients(bg), o.batch_gradients(bo)
    print("masked", masked, "loss", gg.loss, go.loss)
    for f in ("inputs", "targets", "seasonality_slices", "anchor_levels"):
        a, b = getattr(bg, f), getattr(bo, f)
        d = np.abs(a - b).max(axis=-1) if a.ndim > 1 else np.abs(a - b)
        bad = np.nonzero(d > 1e-9)[0]
        print(f, "maxdiff", d.max(), "bad rows", bad[:20])
