"""Small repro for compute-sanitizer runs: one batch_gradients call per profile/precision."""
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
prof, vals, cats = dataset(orc, name, 12, 11)
tr = Trainer((vals, cats), prof, TrainConfig(seed=7, precision=prec, batch_size=16), api=eng)
w = tr.all_windows()[:16]
b = WindowBatch([x[0] for x in w], [x[1] for x in w])
g = tr.batch_gradients(b)
print("loss", g.loss)
print("epoch", tr.train_epoch())
print("val", tr.validate().mean_smape)
