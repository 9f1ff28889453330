"""Try the real NCCL sharded path with two ranks on one GPU (diagnostic; NCCL may refuse
duplicate devices).  Compares the 2-rank epoch loss / validate sMAPE with a 1-rank run."""
import os, sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch.multiprocessing as mp


def worker(rank, world, uid, q):
    from paper_1907_03329_b200 import _native as N
    from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer
    api = N.product_api()
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    vals, cats = api.make_synthetic(41, 64, 88, 4, 0.05)
    cfg = TrainConfig(seed=7, batch_size=256, precision="fp64")
    try:
        tr = Trainer((vals, cats), prof, cfg, api=api, dist=(rank, world, uid))
        out = [tr.train_epoch() for _ in range(2)]
        out.append(tr.validate().mean_smape)
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


if __name__ == "__main__":
    from paper_1907_03329_b200 import _native as N
    from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer
    api = N.product_api()
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    vals, cats = api.make_synthetic(41, 64, 88, 4, 0.05)
    tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=256, precision="fp64"), api=api)
    ref = [tr.train_epoch() for _ in range(2)] + [tr.validate().mean_smape]
    tr.close()
    print("1 rank:", ref, flush=True)
    uid = api.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, uid, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    print("2 ranks:", json.dumps(res), flush=True)
