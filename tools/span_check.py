"""Cross-check the bench's in-graph kernel spans (profile_kernels(2)) against the step-5
debug spans (ESRNN_DEBUG_CLOCKS=1) in one cfg1-shaped run."""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer
api = N.product_api()
prof = FrequencyProfile.defaults(Frequency.Quarterly)
length = prof.min_length + 2 * prof.horizon
vals, cats = api.make_synthetic(41, 1000, length, prof.seasonality_length, 0.05)
tr = Trainer((vals, cats), prof, TrainConfig(batch_size=1000, seed=7, precision='fp32'), api=api)
tr.train_epoch()
tr.profile_kernels(2)
tr.train_epoch()
tr.profile_kernels(2)
for _ in range(3):
    tr.train_epoch()
kt = tr.kernel_times()
print({k: (round(v[0] / 3, 4), v[1] // 3, round(1000 * v[0] / max(v[1], 1), 2)) for k, v in kt.items() if v[1]})
