"""Small repro for compute-sanitizer runs: batch gradients, training epochs (graphs + PDL),
validate / evaluate, the general forward_stack with gradients and the exact-resume state, per
profile / precision; `big` adds a >= 8,192-window step (split weight-gradient tiles).

    compute-sanitizer --tool memcheck python tools/repro_batch.py quarterly fp32 [big]
"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
from conftest import dataset, ORACLE_LIB
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import TrainConfig, Trainer, WindowBatch
eng = N.product_api(); orc = N.NativeApi(ORACLE_LIB)
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
big = len(sys.argv) > 3 and sys.argv[3] == "big"
prof, vals, cats = dataset(orc, name, 160 if big else 12, 11)
bs = 8192 if big else 16
tr = Trainer((vals, cats), prof, TrainConfig(seed=7, precision=prec, batch_size=bs, max_batch_size=max(bs, 2048)),
             api=eng)
w = tr.all_windows()[:bs]
b = WindowBatch([x[0] for x in w], [x[1] for x in w])
g = tr.batch_gradients(b)
print("loss", g.loss)
for _ in range(2):
    print("epoch", tr.train_epoch())
print("val", tr.validate().mean_smape)
print("eval", tr.evaluate(True).mean_smape)
ts = tr.train_state()
tr.set_train_state(ts)
x = np.random.default_rng(0).uniform(-1, 1, (3, 4, prof.input_window + 6))
out, wb, xb = tr.forward_stack(x, np.ones((4, prof.horizon)))
print("stack", float(out.sum()), float(xb.sum()))
# round 2: the inference forward_stack kernel (shared-memory-resident layer weights) and, with
# a penalty, the penalised ES path
print("stack-fast", float(tr.forward_stack(x).sum()))
tp = Trainer((vals, cats), prof, TrainConfig(seed=7, precision=prec, batch_size=bs, max_batch_size=max(bs, 2048),
                                             level_variability_penalty=2.0), api=eng)
print("penalised epoch", tp.train_epoch())
