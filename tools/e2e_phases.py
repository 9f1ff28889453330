"""Time the phases of one e2e step (construct / epoch / validate / destroy) on cuda:0."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer

api = N.product_api()
prof = FrequencyProfile.defaults(Frequency.Quarterly)
vals, cats = api.make_synthetic(41, 1000, 88, 4, 0.05)
cfg = TrainConfig(seed=7, batch_size=1000, precision="fp32", max_batch_size=2048)
for it in range(6):
    t = [time.perf_counter()]
    tr = Trainer((vals, cats), prof, cfg, api=api); t.append(time.perf_counter())
    tr.train_epoch(); t.append(time.perf_counter())
    tr.train_epoch(); t.append(time.perf_counter())
    tr.validate(); t.append(time.perf_counter())
    tr.close(); t.append(time.perf_counter())
    d = [1000 * (b - a) for a, b in zip(t, t[1:])]
    print("create %.2f epoch1 %.2f epoch2 %.2f validate %.2f destroy %.2f ms" % tuple(d), flush=True)
