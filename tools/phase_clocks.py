"""Print per-phase clock64 stamps of k_tile tile 0 (ESRNN_DEBUG_CLOCKS=1, no graphs)."""
import os, sys
from pathlib import Path
os.environ["ESRNN_DEBUG_CLOCKS"] = "1"
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer
api = N.product_api()
freq = Frequency[sys.argv[1]] if len(sys.argv) > 1 else Frequency.Quarterly
prof = FrequencyProfile.defaults(freq)
n, B = (1000, 1000) if freq == Frequency.Quarterly else ((23000, 2048) if freq == Frequency.Yearly else (48000, 2048))
length = prof.min_length + 2 * prof.horizon
vals, cats = api.make_synthetic(41, n, length, prof.seasonality_length, 0.05)
tr = Trainer((vals, cats), prof, TrainConfig(batch_size=B, seed=7, use_graphs=os.environ.get('GRAPHS') == '1', max_batch_size=max(B, 2048), precision='fp32'), api=api)
for _ in range(2):
    tr.train_epoch()
