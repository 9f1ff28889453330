import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200.trainer import *
api = N.product_api(); prof = FrequencyProfile.defaults(Frequency.Monthly)
v, c = api.make_synthetic(41, 64, 108, 12, 0.05)
tr = Trainer((v, c), prof, TrainConfig(seed=7, batch_size=64, precision="fp32"), api=api)
x = np.random.default_rng(1).uniform(0.5, 1.5, size=(72, 2048, 30))
for _ in range(2): tr.forward_stack(x)
print(tr.last_device_ms())
