"""cProfile of the e2e step's host side (Trainer construction + epoch + validate + destroy)."""
import cProfile, pstats, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer

api = N.product_api()
prof = FrequencyProfile.defaults(Frequency.Quarterly)
vals, cats = api.make_synthetic(41, 1000, 88, 4, 0.05)
cfg = TrainConfig(seed=7, batch_size=1000, precision="fp32", max_batch_size=2048)


def step():
    tr = Trainer((vals, cats), prof, cfg, api=api)
    tr.train_epoch()
    tr.validate()
    tr.close()


for _ in range(5):
    step()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
for _ in range(20):
    step()
dt = (time.perf_counter() - t0) / 20
pr.disable()
print(f"e2e step {dt * 1e3:.3f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
